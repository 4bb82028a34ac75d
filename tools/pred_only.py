"""cfg #3 predictor launches only (profiling target): 10M forest queries, 2 launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
import paper_2405_05465_b200 as ssg
ssg.init(0)
r = bench.predictor_bench(torch, dev, 10_000_000, 1, 1)
print(r["value"], r["e2e"], r["roofline"].get("compulsory_bytes_per_query"))
