"""C4 'down' shape (4096 x 14336 f32): default chunked variant vs an SCB_VARIANT override."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_01799_b200 as sc
from paper_2410_01799_b200.batch import mistral_jobs, mistral_matrix
eng = sc.Engine(0)
j = mistral_jobs()[6]
a = mistral_matrix(j)
for _ in range(3):
    dec, rep, _ = eng.run(a, sc.DecomposeConfig(width=64, search=sc.SearchConfig(seed=j.seed)), dtype="f32")
    print(os.environ.get("SCB_VARIANT", "default"), "kernel_ms", round(rep.kernel_ms, 2), "passes", rep.passes,
          "us/pass", round(rep.kernel_ms * 1e3 / rep.passes, 1), "rel", rep.final_residual_norm / rep.input_norm, flush=True)
