"""Summarise one round's ncu captures into profiles/<tag>/ (tracked).

usage: python scripts/ncu_summary.py --rep gpurun_out/X.ncu-rep --out profiles/r02/X.txt --desc "..." \
           --cuts N [--launches gpurun_out/launches.csv] [--traffic]
outputs: the summary text, launches.csv / launches_summary.txt beside it, and with --traffic
         profiles/latest_kernel_traffic.json (read by bench.py for roofline.traffic when its
         cuts per launch match the bench width)
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

FULL_METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("lts__t_bytes.sum", "L2 bytes (all)"),
    ("lts__t_sectors.sum", "L2 sectors (all, x32 B)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "SMEM wavefronts"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic SMEM/block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def launches(src, dst, desc):
    lines = open(src).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}[r[ui]]
        k = r[ki]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    shutil.copy(src, os.path.join(dst, "launches.csv"))
    with open(os.path.join(dst, "launches_summary.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list of\n#   {desc}\n"
                f"# per-launch times are cold-cache and serialised: compare SHARES, not absolutes\n")
        f.write(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{n:8d} {t:10.3f} {t / tot:7.2%}  {k}\n")
    return agg


def full(rep, out_txt, desc, cuts, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {name: (v[h.index(name)], u[h.index(name)]) for name, _ in FULL_METRICS if name in h}
    stalls = sorted(((x, float(v[i] or 0)) for i, x in enumerate(h)
                     if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio")),
                    key=lambda t: -t[1])[:10]
    with open(out_txt, "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 of\n#   {desc}\n")
        f.write(f"kernel: {v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'}\n")
        f.write(f"cuts per launch              {cuts:>18d}\n")
        for name, label in FULL_METRICS:
            if name in get:
                f.write(f"{label:28s} {get[name][0]:>18s} {get[name][1]}\n")
        f.write("\ntop stall reasons (warps per issue-active cycle):\n")
        for x, val in stalls:
            f.write(f"  {x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {val:.3f}\n")

    def num(name, to):
        val, unit = get[name]
        val = float(val.replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6,
                "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0, "second": 1.0}[unit]
        return val * mult / to

    traffic = {
        "kernel": desc,
        "cuts_per_launch": cuts,
        "dram_bytes_per_launch": num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1),
        "dram_read_bytes": num("dram__bytes_read.sum", 1),
        "dram_write_bytes": num("dram__bytes_write.sum", 1),
        "duration_s_under_ncu": num("gpu__time_duration.sum", 1),
        "l2_bytes_per_launch": (float(get["lts__t_sectors.sum"][0].replace(",", "")) * 32.0
                                if "lts__t_sectors.sum" in get else None),
        "source": os.path.relpath(out_txt, ROOT),
    }
    if traffic_json:
        with open(traffic_json, "w") as f:
            json.dump(traffic, f, indent=1)
    return traffic


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True, help="gpurun_out/<name>.ncu-rep (--set full, one sweep_kernel launch)")
    ap.add_argument("--out", required=True, help="profiles/<round>/<name>.txt")
    ap.add_argument("--desc", required=True)
    ap.add_argument("--cuts", type=int, required=True)
    ap.add_argument("--launches", default="", help="gpurun_out/<launch list>.csv")
    ap.add_argument("--traffic", action="store_true", help="also write profiles/latest_kernel_traffic.json")
    args = ap.parse_args()
    dst = os.path.dirname(os.path.abspath(args.out))
    os.makedirs(dst, exist_ok=True)
    if args.launches:
        launches(args.launches, dst, args.desc)
        print(open(os.path.join(dst, "launches_summary.txt")).read())
    tr = full(args.rep, args.out, args.desc, args.cuts,
              os.path.join(ROOT, "profiles", "latest_kernel_traffic.json") if args.traffic else None)
    print(open(args.out).read())
    print(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main()
