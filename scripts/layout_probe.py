"""Is the 4096^2 f32 64-cut time a function of where the engine's buffers land?
Runs the same decomposition on several engines created in one process (some
alive at the same time) and prints kernel ms per run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import _native as N

if os.environ.get("PROBE_LIB"):
    N.LIB_PATH = os.environ["PROBE_LIB"]

MODE = os.environ.get("PROBE_MODE", "plain")  # plain | torch | torchbuf | torchflush
flush = None
if MODE != "plain":
    import torch
    torch.cuda.init()
    if MODE in ("torchbuf", "torchflush"):
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print("mode", MODE, flush=True)
a = sc.fill_normal(1, 4096 * 4096, np.float32).reshape(4096, 4096)
cfg = sc.DecomposeConfig(width=64, search=sc.SearchConfig(seed=1))


def runs(eng, tag, k=3):
    ms = []
    for _ in range(k):
        if MODE == "torchflush":
            flush.zero_()
            torch.cuda.synchronize()
        dec, rep, _ = eng.run(a, cfg, dtype="f32")
        ms.append(round(rep.kernel_ms, 2))
    print(tag, ms, flush=True)


if os.environ.get("PROBE_SHIFTS"):  # one engine, the arena carve shifted per run
    e = sc.Engine(0)
    for spec in os.environ["PROBE_SHIFTS"].split(";"):
        os.environ["SCB_ARENA_SHIFT"] = "0"
        os.environ["SCB_SYNC_SHIFT"] = "0"
        os.environ["SCB_SLOT_SHIFT"] = "0"
        os.environ["SCB_TB_SHIFT"] = "0"
        os.environ["SCB_ZS_SHIFT"] = "0"
        for kv in spec.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
        runs(e, spec, 2)
    sys.exit(0)
e1 = sc.Engine(0)
runs(e1, "e1")
e2 = sc.Engine(0)
runs(e2, "e2 (e1 alive)")
runs(e1, "e1 again")
del e1
e3 = sc.Engine(0)
runs(e3, "e3 (e1 freed)")
del e2, e3
for i in range(4):
    e = sc.Engine(0)
    runs(e, f"fresh {i}", 1)
    del e
