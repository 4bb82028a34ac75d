import json, sys, os
sys.path.insert(0, os.getcwd())
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
from oracle import ref
ssg.init(0)
spec, dev = catalog.MODELS["llama2_7b"], catalog.DEVICES["a100_80g"]
want = json.loads(ref.train(spec, dev, [1], "forest", 42))
got = json.loads(ssg.Estimator.train(spec, dev, [1], "forest", seed=42).to_json())
out = open("gpurun_out/dbg_train.txt", "w")
for k in want["ops"]:
    a, b = want["ops"][k], got["ops"][k]
    for field in a:
        if field != "regressor" and a[field] != b[field]:
            print(k, "field", field, a[field], b[field], file=out)
    ra, rb = a["regressor"], b["regressor"]
    for f in ("y_lo", "y_hi", "num_features"):
        if ra[f] != rb[f]: print(k, f, ra[f], rb[f], file=out)
    for t, (ta, tb) in enumerate(zip(ra["trees"], rb["trees"])):
        if ta != tb:
            print(k, "tree", t, file=out)
            for f in ("feature", "threshold", "left", "right", "leaf_weights"):
                print("  ", f, "\n    ref", ta[f], "\n    ssg", tb[f], file=out)
            break
out.close()
import time
for model, d, tps in (("llama2_70b", "h100_80g", [4]), ("qwen_72b", "a100_80g", [1, 2, 4])):
    t0 = time.time(); ssg.Estimator.train(catalog.MODELS[model], catalog.DEVICES[d], tps, "forest", seed=7); t1 = time.time()
    ref.train(catalog.MODELS[model], catalog.DEVICES[d], tps, "forest", 7); t2 = time.time()
    print("train %s %s: ssg %.2f s, reference %.2f s" % (model, tps, t1 - t0, t2 - t1), flush=True)
