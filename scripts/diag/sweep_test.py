import sys, json; sys.path.insert(0, ".")
import bench, paper_2410_07531_b200 as rgo
print(json.dumps(bench.bench_seq_sweep(rgo, 0, 1, [1024, 2048, 4096, 8192])))
