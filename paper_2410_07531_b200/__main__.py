"""Command line for the dropout path -- the `maskgen` and `verify`
subcommands of the reference CLI (proj/tools/rgo_cli.cpp:147-166, 230-247),
same options, defaults, output and exit codes (std::invalid_argument -> 2,
other failures -> 1).  The reference's model/sweep/capacity/whatif
subcommands drive its analytical limiter model, which is out of this
build's scope.

    python -m paper_2410_07531_b200 maskgen --b 1 --nh 8 --sq 512 --p 0.9 --seed 42 --out m.rngm
    python -m paper_2410_07531_b200 verify --rounds 7
"""
from __future__ import annotations

import argparse
import sys


def _u64(s: str) -> int:
    v = int(s, 0)
    if not 0 <= v < (1 << 64):
        raise argparse.ArgumentTypeError("expected a 64-bit unsigned integer")
    return v


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="rgo", description="B200 dropout-RNG pipeline (maskgen / verify)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    m = sub.add_parser("maskgen", help="write a dropout mask file")
    m.add_argument("--b", type=int, required=True, help="batch size")
    m.add_argument("--nh", type=int, required=True, help="number of heads")
    m.add_argument("--sq", type=int, required=True, help="sequence length")
    m.add_argument("--p", type=float, required=True, help="keep probability")
    m.add_argument("--seed", type=_u64, required=True, help="64-bit seed")
    m.add_argument("--base-offset", type=_u64, default=0, help="counter offset")
    m.add_argument("--rounds", type=int, default=7, help="Philox rounds")
    m.add_argument("--workers", type=int, default=0, help="devices to shard over (0 = all; bytes do not change)")
    m.add_argument("--out", required=True, help="output mask file")
    v = sub.add_parser("verify", help="fused vs decoupled dropout equivalence suite")
    v.add_argument("--rounds", type=int, default=7, help="Philox rounds")
    args = ap.parse_args(argv)

    from . import mask as M
    from . import ref_attention as A
    try:
        if args.cmd == "maskgen":
            lay = M.MaskLayout(args.b, args.nh, args.sq, args.seed, args.base_offset)
            mk = M.generate_mask(lay, M.KeepThreshold(args.p), args.rounds, args.workers)
            M.save_mask(mk, args.out)
            return 0
        results = A.run_equiv_suite(A.default_equiv_grid(), args.rounds)
        bad = 0
        for r in results:
            c = r.c
            print(f"{'ok' if r.bitwise_equal else 'FAIL':<4} slices={c.slices} sq={c.seq} dh={c.head_dim} "
                  f"seed={c.seed} p={c.p:.2f}")
            bad += 0 if r.bitwise_equal else 1
        print(f"{len(results)} cases, {bad} mismatches")
        return 1 if bad else 0
    except ValueError as e:  # std::invalid_argument
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001  (rgo_cli.cpp:267-270)
        print(f"internal error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
