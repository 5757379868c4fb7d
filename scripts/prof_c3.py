"""Phase split of the order-3 C3 pass (needs an SCB_PROFILE=1 build; engine option profile=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01799_b200 import _native as N
if os.environ.get("SCB_LIB"):  # an SCB_PROFILE=1 build
    N.LIB_PATH = os.environ["SCB_LIB"]
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import workloads as wl
eng = sc.Engine(0, profile=1)
img = wl.c3_blob_image()
for w in (4, 64):
    dec, rep, _ = eng.run(img, sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=2)), dtype="f32")
    print("w", w, "kernel_ms", rep.kernel_ms, "passes", rep.passes, "us/pass", rep.kernel_ms * 1e3 / rep.passes, flush=True)
a = img.reshape(4000, 9000)
dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=64, search=sc.SearchConfig(seed=2)), dtype="f32")
print("matrix view 4000x9000 w 64 kernel_ms", rep.kernel_ms, "passes", rep.passes, "us/pass", rep.kernel_ms * 1e3 / rep.passes)
