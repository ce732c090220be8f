"""The maskgen / verify command line (rgo_cli.cpp:147-166, 230-247)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2410_07531_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=300)


def test_invalid_arguments_exit_2(tmp_path):
    # validation precedes any device work (generate_mask, mask.hpp:142-155)
    r = cli("maskgen", "--b", "1", "--nh", "1", "--sq", "8", "--p", "0.9", "--seed", "1", "--rounds", "17",
            "--out", str(tmp_path / "m"))
    assert r.returncode == 2 and "rounds" in r.stderr
    r = cli("maskgen", "--b", "0", "--nh", "1", "--sq", "8", "--p", "0.9", "--seed", "1", "--out", str(tmp_path / "m"))
    assert r.returncode == 2 and "zero elements" in r.stderr
    r = cli("maskgen", "--b", "1", "--nh", "1", "--sq", "8", "--p", "1.5", "--seed", "1", "--out", str(tmp_path / "m"))
    assert r.returncode == 2


@pytest.mark.gpu
def test_maskgen_file_matches_oracle(tmp_path):
    out = tmp_path / "o.rngm"
    r = cli("maskgen", "--b", "1", "--nh", "8", "--sq", "512", "--p", "0.9", "--seed", "42", "--rounds", "10",
            "--out", str(out))
    assert r.returncode == 0, r.stderr
    blob = out.read_bytes()
    assert len(blob) == 40 + 8 * 512 * 512 // 8 and blob[:4] == b"RNGM"
    want = oracle.generate_mask(1, 8, 512, 42, 0, 0.9, 10)
    assert np.array_equal(np.frombuffer(blob[40:], np.uint8), want)


@pytest.mark.gpu
def test_verify_suite_passes():
    r = cli("verify", "--rounds", "7")
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "16 cases, 0 mismatches" and all(l.startswith("ok") for l in lines[:-1])
