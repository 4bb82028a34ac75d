"""One cfg #2 simulation through ssg_simulate_run (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
est = ssg.Estimator.train(catalog.MODELS["llama2_70b"], catalog.DEVICES["h100_80g"], [4], "interp", seed=0)
pre, dec = ssg.synth_trace(catalog.zipf_histogram(), 10000, 42)
cl = catalog.cluster_doc("llama2_70b", "h100_80g", tp=4, policy="sarathi_serve", max_batch_size=128, chunk_size=512)
arr = ssg.poisson_arrivals(10000, 10.0, 0)
run = ssg.simulate_run(cl, est, np.arange(10000), arr, pre, dec)
print("span", run.report.simulated_span)
