"""C3 (order-3 blob image) with a small width: ncu target for the order-k pass.
usage: c3_small.py [width] [repeats]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import workloads as wl
eng = sc.Engine(0)
img = wl.c3_blob_image()
w = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    dec, rep, _ = eng.run(img, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=2)), dtype="f32")
    print("w", w, "kernel_ms", round(rep.kernel_ms, 2), "passes", rep.passes, "us/pass",
          round(rep.kernel_ms * 1e3 / rep.passes, 1), "2ph", os.environ.get("SCB_2PH", "auto"), flush=True)
