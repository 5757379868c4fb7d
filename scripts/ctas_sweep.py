"""Pass time vs grid size (SCB_CTAS caps G); one process per setting.
CS_SHAPE="m,n,width,seed" (default C1: 1024,1024,256,0)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2410_01799_b200 as sc\n"
        "m, n, w, sd = (int(x) for x in %r.split(','))\n"
        "eng = sc.Engine(0); a = sc.fill_normal(sd, m * n, np.float32).reshape(m, n)\n"
        "cfg = sc.DecomposeConfig(width=w, search=sc.SearchConfig(seed=sd))\n"
        "eng.run(a, sc.DecomposeConfig(width=8), dtype='f32')\n"
        "ts = [eng.run(a, cfg, dtype='f32')[1] for _ in range(3)]\n"
        "r = min(ts, key=lambda r: r.kernel_ms)\n"
        "print(round(r.kernel_ms, 2), 'ms', round(r.kernel_ms * 1e3 / r.passes, 2), 'us/pass', r.passes)\n") % (
    ROOT, os.environ.get("CS_SHAPE", "1024,1024,256,0"))
for g in sys.argv[1:] or ["16", "32", "48", "64", "96", "128"]:
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SCB_CTAS=g), capture_output=True, text=True)
    print("G<=" + g, out.stdout.strip(), out.stderr.strip()[-200:], flush=True)
