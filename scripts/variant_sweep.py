"""C1 (1024^2 f32, w=256) and 1024x4096 pass time per kernel variant (SCB_VARIANT), one process each."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, paper_2410_01799_b200 as sc\n"
        "m, n = %s\n"
        "eng = sc.Engine(0); a = sc.fill_normal(0, m * n, np.float32).reshape(m, n)\n"
        "cfg = sc.DecomposeConfig(width=128, search=sc.SearchConfig(seed=0))\n"
        "eng.run(a, sc.DecomposeConfig(width=4), dtype='f32')\n"
        "r = min((eng.run(a, cfg, dtype='f32')[1] for _ in range(2)), key=lambda r: r.kernel_ms)\n"
        "print(round(r.kernel_ms, 2), 'ms', round(r.kernel_ms * 1e3 / r.passes, 2), 'us/pass', r.passes)\n")
for shape in ["1024, 1024", "1024, 4096"]:
    for v in ["", "8,1,4", "8,2,2", "16,2,2", "16,2,1", "8,4,2", "8,4,1"]:
        env = dict(os.environ)
        if v:
            env["SCB_VARIANT"] = v
        out = subprocess.run([sys.executable, "-c", code % (ROOT, shape)], env=env, capture_output=True, text=True)
        print(shape, v or "default", out.stdout.strip(), out.stderr.strip()[-150:], flush=True)
