"""Throughput of independent decompositions co-scheduled on one GPU: K engines (own
contexts/streams) in K host threads, each grid capped at G / K CTAs (SCB_CTAS), vs one
engine with the whole GPU run K times back to back."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_01799_b200 as sc
shape = tuple(int(x) for x in os.environ.get("CS_SHAPE", "4096,4096").split(","))
W = int(os.environ.get("CS_W", 32))
K = int(os.environ.get("CS_K", 2))
a = sc.fill_normal(1, shape[0] * shape[1], np.float32).reshape(shape)
cfg = sc.DecomposeConfig(width=W, search=sc.SearchConfig(seed=1))
engs = [sc.Engine(0) for _ in range(K)]
for e in engs:
    e.run(a, sc.DecomposeConfig(width=2, search=sc.SearchConfig(seed=1)), dtype="f32")
def work(e, out):
    out.append(e.run(a, cfg, dtype="f32")[1])
t0 = time.perf_counter()
res = []
ths = [threading.Thread(target=work, args=(e, res)) for e in engs]
[t.start() for t in ths]
[t.join() for t in ths]
dt = time.perf_counter() - t0
print(f"{os.environ.get('SCB_CTAS', 'all')} CTAs x {K} concurrent {shape} w={W}: {K * W / dt:.1f} cuts/s "
      f"(kernel ms {[round(r.kernel_ms, 1) for r in res]}, us/pass {[round(r.kernel_ms * 1e3 / r.passes, 1) for r in res]})", flush=True)
