"""Delta-pass policy sweep: SCB_DELTA_DIV (a delta pass runs when the flipped
t columns are <= n / DIV) and SCB_DELTA_REFRESH (dense refresh every R sweeps).
Prints kernel ms and whether every term's signs match the default policy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc

shapes = [(4096, 4096, 64, 1), (1024, 1024, 256, 0)]
if os.environ.get("DS_C3"):  # config 3 (order 3) instead: the blob image, search seed 2
    shapes = [("c3", None, int(os.environ.get("DS_W", 128)), 2)]
pol = [(32, 16), (16, 16), (8, 16), (4, 16), (2, 16), (32, 32), (8, 32), (8, 64), (4, 64)]
if os.environ.get("DS_POL"):
    pol = [tuple(int(x) for x in q.split(":")) for q in os.environ["DS_POL"].split(",")]
eng = sc.Engine(0)
for m, n, w, seed in shapes:
    if m == "c3":
        from paper_2410_01799_b200 import workloads as wl
        a = wl.c3_blob_image()
    else:
        a = sc.fill_normal(1 if seed else 0, m * n, np.float32).reshape(m, n)
    cfg = sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=seed))
    base = None
    for div, ref in pol:
        os.environ["SCB_DELTA_DIV"], os.environ["SCB_DELTA_REFRESH"] = str(div), str(ref)
        ms = []
        for _ in range(2):
            dec, rep, _ = eng.run(a, cfg, dtype="f32")
            ms.append(rep.kernel_ms)
        sig = [f.copy() for f in dec.factors]
        if base is None:
            base = sig
        same = all((x == y).all() for x, y in zip(sig, base))
        print(f"{a.shape} w={w} div={div} refresh={ref}: {min(ms):.2f} ms passes {rep.passes} "
              f"same_signs={same} rel={rep.final_residual_norm / rep.input_norm:.9f}", flush=True)
