"""Times k_predict on the cfg #3 query mix (diagnostic)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2405_05465_b200 as ssg
ssg.init(0)
dev = torch.device("cuda", 0)
nq = int(os.environ.get("NQ", "10000000"))
r = bench.predictor_bench(torch, dev, nq, int(os.environ.get("STEPS", "3")), 2)
print(json.dumps(r, indent=1))
