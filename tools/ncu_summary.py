"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md> [label]
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic_key]

`launches`: per-kernel launch counts, total and mean device time, and share
of all kernel time (cold-cache, serialised: compare SHARES with bench.py's
kernel_share_of_step, not absolutes).
`full`: the headline metrics of one --set full capture (duration, DRAM
bytes read/written = traffic, DRAM throughput, SM active, occupancy,
registers, warp stall breakdown) and, with a key, records the per-launch
traffic into profiles/traffic.json for bench.py's roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    n = name.split("(")[0]
    if "sweep_kernel" in name:
        import re
        m = re.search(r"Cfg<(\w+), \(int\)(\d), \(int\)(\d), \(int\)(\d), \(int\)(\d), \(int\)(\d)", name)
        if m:
            t, nd, sh, rr, q, s = m.groups()
            return "sweep_kernel<%s,%dD,%s,q=%s,stages=%s>" % (t, int(nd), "star" if sh == "0" else "box", q, s)
    return n.replace("void ", "")


def launches(path, out, label=""):
    rows = [l for l in open(path) if not l.startswith("==")]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    agg = OrderedDict()
    total = 0.0
    n = 0
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"])
        if r.get("Metric Unit") == "us":
            v *= 1e3
        elif r.get("Metric Unit") == "ms":
            v *= 1e6
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
        n += 1
    lines = ["# ncu launch list summary %s" % label, "",
             "Source: `%s` (`ncu --metrics gpu__time_duration.sum --clock-control none`)." % os.path.basename(path),
             "Per-launch times are cold-cache and serialised; compare the SHARE with bench.py's",
             "`roofline.kernel_share_of_step`.", "",
             "| kernel | launches | total ms | mean us | share of kernel time |", "|---|---:|---:|---:|---:|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append("| `%s` | %d | %.3f | %.2f | %.1f%% |" % (k, c, t / 1e6, t / c / 1e3, 100 * t / total))
    lines.append("")
    lines.append("Total: %d launches, %.3f ms of kernel time." % (n, total / 1e6))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}

    def g(name):
        x = d.get(name)
        return (x[0], x[1]) if x else ("-", "")
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "sm__cycles_active.min",
            "sm__cycles_active.max", "gpc__cycles_elapsed.max", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"]
    kname = ""
    for row in r[2:3]:
        kname = row[h.index("Kernel Name")] if "Kernel Name" in h else ""
    lines = ["# ncu --set full summary", "", "Report: `%s`" % os.path.basename(rep), "",
             "Kernel: `%s`" % short(kname), "", "| metric | value | unit |", "|---|---:|---|"]
    for w in want:
        val, unit = g(w)
        lines.append("| `%s` | %s | %s |" % (w, val, unit))
    stalls = [(k, float(v or 0)) for k, (v, _) in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(s for _, s in stalls) or 1.0
    lines += ["", "Warp stall samples (share):", ""]
    for k, s in sorted(stalls, key=lambda kv: -kv[1])[:8]:
        lines.append("- `%s`: %.1f%%" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * s / tot))
    try:
        rd_b = float(g("dram__bytes_read.sum")[0])
        wr_b = float(g("dram__bytes_write.sum")[0])
        unit = g("dram__bytes_read.sum")[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        traffic = (rd_b + wr_b) * scale
        lines += ["", "traffic (dram read + write per launch): %.4e bytes" % traffic]
        if key:
            tp = os.path.join(ROOT, "profiles", "traffic.json")
            t = json.load(open(tp)) if os.path.exists(tp) else {}
            t[key] = traffic
            json.dump(t, open(tp, "w"), indent=1, sort_keys=True)
    except ValueError:
        pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
