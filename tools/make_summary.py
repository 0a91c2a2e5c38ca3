"""Write profiles/<tag>_summary.md from a bench line, launch lists and one ncu --set full report.

usage: python tools/make_summary.py TAG BENCH.json REF.json CFG2_LAUNCHES.csv CFG4_LAUNCHES.csv REPORT.ncu-rep NOTES.md
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_profiles import launch_shares, stall_breakdown  # noqa: E402

tag, bench, ref, l2, l4, rep, notes = sys.argv[1:8]
d = json.loads(open(bench).read().strip().splitlines()[-1])
r = json.loads(open(ref).read().strip().splitlines()[-1])
print(f"# ncu summary, {tag}\n")
print("All captures: one B200, `ncu --clock-control none`; launch lists are cold-cache and serialised (compare shares,")
print("not absolute times).  Raw CSVs and the bench lines are beside this file.\n")
print("## Bench (`python bench.py`, default steps)\n")
print("| workload | ms / step | DOF-sweeps/s | e2e | CG roofline frac | solve us | traffic / algorithmic |")
print("|---|---|---|---|---|---|---|")
print(f"| cfg2 (headline) | {d['ms_per_step']:.3f} | {d['value']:.3e} | {d['e2e']['value']:.3e} | "
      f"{d['roofline']['frac']:.3f} (latency bound) | {d['roofline']['kernel_us']:.1f} | - |")
for k, v in d["secondary"].items():
    rf = v["roofline"]
    tr = rf["traffic"] / rf["algorithmic_bytes_per_launch"] if rf["traffic"] else float("nan")
    print(f"| {k} | {v['ms_per_step']:.1f} | {v['value']:.3e} | {v['e2e']['value']:.3e} | {rf['frac']:.3f} | "
          f"{rf['kernel_us']:.0f} | {tr:.3f} |")
print(f"\nReference arm (`--impl reference`: the unmodified `sisdc.mlsdc.run_mlsdc` from `oracle/_ref`, SuperLU, "
      f"{r['cpu_baseline']['cores']} host threads available): {r['ms_per_step']:.1f} ms per cfg2 step = {r['value']:.3e} "
      f"DOF-sweeps/s -> {d['e2e']['value'] / r['value']:.1f}x end to end.\n")
for name, path in (("cfg2 (`bench.py --no-2d --steps 3 --warmup 1`)", l2),
                   ("cfg4 (`bench.py --workload cfg4 --no-cfg5 --steps 2 --warmup 1`; includes the bench's roofline solves)", l4)):
    print(f"## Launch list, {name}\n")
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    sh, tot = launch_shares(path)
    for k, n, t, m, p in sh[:16]:
        print(f"| {k} | {n} | {t:.1f} | {m:.2f} | {p:.1f}% |")
    print(f"\ntotal device time {tot:.1f} us\n")
print("## k2_cgf<4,1,0>, ncu --set full (`tools/cg2_one.py cfg4 7 1`, 24 iterations)\n\n```")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
for k in want:
    if k in h:
        print(f"{k}: {v[h.index(k)]} {u[h.index(k)]}")
print("```\n\n## Stall reasons (all samples)\n")
for k, vv in stall_breakdown(rep):
    print(f"- {k}: {vv}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
print("\n## Hottest source lines (`tools/ncu_lines.py`)\n\n```")
print(subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_lines.py"),
                      "/tmp/_src.csv", "14"], capture_output=True, text=True).stdout)
print("```\n")
print(open(notes).read())
