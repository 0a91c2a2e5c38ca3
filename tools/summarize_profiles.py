"""Summarise ncu outputs (launch list CSV + one --set full report) into profiles/."""
import collections, csv, io, json, subprocess, sys


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] in ("usecond", "us"):
            v *= 1e3
        elif d["Metric Unit"] in ("msecond", "ms"):
            v *= 1e6
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    return [(k, n, t / 1e3, t / n / 1e3, 100 * t / tot) for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])], tot / 1e3


def report_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__block_size", "launch__grid_size", "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    res = []
    for v in vals:
        d = dict(zip(hdr, v))
        res.append({k: (d.get(k), units[hdr.index(k)] if k in hdr else None) for k in want if k in hdr})
    return res


def stall_breakdown(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    agg = collections.Counter()
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr) - 1:
            d = dict(zip(hdr, r))
            for h in hdr:
                if h.startswith("stall_") and "Not Issued" not in h:
                    try:
                        agg[h] += float(d[h])
                    except ValueError:
                        pass
    tot = sum(agg.values()) or 1
    return [(k, round(100 * v / tot, 1)) for k, v in agg.most_common(10)]


if __name__ == "__main__":
    launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [f"# ncu summary, {tag}", "", "## Launch list (bench.py, cold-cache serialised: compare shares)", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    sh, tot = launch_shares(launches)
    for k, n, t, m, p in sh:
        lines.append(f"| {k} | {n} | {t:.1f} | {m:.2f} | {p:.1f}% |")
    lines += ["", f"total device time {tot:.1f} us", "", "## k_cg1d, ncu --set full (2 launches)", "", "```"]
    for m in report_metrics(rep):
        lines.append(json.dumps(m))
    lines += ["```", "", "## Stall reasons (all samples, SASS source page)", ""]
    for k, v in stall_breakdown(rep):
        lines.append(f"- {k}: {v}%")
    print("\n".join(lines))
