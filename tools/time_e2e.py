"""Times the e2e ssg_search_shard call on the cfg #4 config (diagnostic; SSG_TIMING=1 prints its phases)."""
import os, sys, time, tempfile
sys.path.insert(0, os.getcwd())
import paper_2405_05465_b200 as ssg
from paper_2405_05465_b200 import catalog
ssg.init(0)
d = tempfile.mkdtemp(); path = catalog.write_search_config(d)
for i in range(3):
    t0 = time.time(); r = ssg.search_shard(path, 0, 1); t1 = time.time()
    print("e2e search_shard %.3f s" % (t1 - t0), flush=True)
