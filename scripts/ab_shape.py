"""Same-box A/B of two engine builds on one C4 job (AB_JOB index, default 6 = down)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200 import _native as N
from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix
libs = [os.environ["SCB_LIB_A"]] + os.environ["SCB_LIB_B"].split(",")
j = mistral_jobs()[int(os.environ.get("AB_JOB", 6))]
a = mistral_matrix(j)
cfg = sc.DecomposeConfig(width=int(os.environ.get("AB_W", 64)), search=sc.SearchConfig(seed=j.seed))
ALL = dict(N.SIGNATURES)
for rnd in range(int(os.environ.get("AB_ROUNDS", 2))):
    for path in libs:
        probe = ctypes.CDLL(path)
        N.SIGNATURES = {k: v for k, v in ALL.items() if hasattr(probe, k)}
        N._lib = None
        N.LIB_PATH = path
        eng = sc.Engine(0)
        dec, rep, _ = eng.run(a, cfg, dtype="f32")
        print(j.name, os.path.basename(path), "kernel_ms %.2f" % rep.kernel_ms, "passes", rep.passes, flush=True)
        del eng
