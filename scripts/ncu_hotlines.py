"""Per-CUDA-source-line warp-stall samples of an ncu --set full --import-source capture
(the kernel built with -lineinfo): the top lines with their two largest stall reasons.
usage: python scripts/ncu_hotlines.py gpurun_out/X.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, fname, cur = None, None, None
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ia, ie = 4, hdr.index("Instructions Executed")
        reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]), r[1].strip()[:72])
        continue
    if cur is None:
        continue
    try:
        s, e = float(r[ia] or 0), float(r[ie] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += s
    a[1] += e
    for i, h in reasons:
        try:
            a[2][h[6:]] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1.0
tote = sum(v[1] for v in agg.values()) or 1.0
reasons_tot = collections.Counter()
for v in agg.values():
    reasons_tot.update(v[2])
rt = sum(reasons_tot.values()) or 1.0
print(f"# {rep}: warp-stall samples per CUDA source line (top {top}); stall reasons overall:")
print("#   " + "  ".join(f"{n} {100 * c / rt:.1f}%" for n, c in reasons_tot.most_common(8)))
print(f"{'samples':>8} {'instr':>7}  line  source  [top stall reasons]")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    r2 = " ".join(f"{n}:{100 * c / max(1, v[0]):.0f}%" for n, c in v[2].most_common(2))
    print(f"{100 * v[0] / tot:7.2f}% {100 * v[1] / tote:6.2f}%  {k[0][:14]}:{k[1]}  {k[2]}  [{r2}]")
