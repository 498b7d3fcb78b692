"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py rep  <file.ncu-rep> <out.md> [--traffic <cfg> <alg_bytes>]
  python tools/ncu_summary.py list <launches.csv> <out.md>

`rep` writes the headline sections of a `ncu --set full` capture (one kernel
launch) as markdown; with --traffic it also writes profiles/traffic_<cfg>.json
(dram bytes per launch, read by bench.py for roofline.traffic).  `list`
aggregates a `--metrics gpu__time_duration.sum` launch list per kernel (cold
cache, serialised: shares, not absolute step times)."""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
           "L2 Cache Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Issue Slots Busy", "Executed Instructions", "Warp Cycles Per Issued Instruction",
           "Eligible Warps Per Scheduler", "Achieved Occupancy", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "SM Frequency"]
RAW = [r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$",
       r"^l1tex__data_pipe_lsu_wavefronts\.sum\.pct_of_peak_sustained_elapsed$",
       r"^l1tex__data_pipe_tc_wavefronts_mem_shared\.sum$",
       r"^l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$",
       r"^l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld\.sum$",
       r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$",
       r"^sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_elapsed$",
       r"^l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld\.sum$",
       r"^l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st\.sum$"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(v.replace(",", "")) * mult.get(unit, 1)


def rep_summary(rep, out_md, traffic=None):
    r = ncu_csv(rep, "details")
    h = r[0]
    name = r[1][h.index("Kernel Name")]
    seen = {}
    for x in r[1:]:
        if x[h.index("ID")] != r[1][h.index("ID")]:
            break
        m = x[h.index("Metric Name")]
        if m in DETAILS and m not in seen:
            seen[m] = f"{x[h.index('Metric Value')]} {x[h.index('Metric Unit')]}".strip()
    raw = ncu_csv(rep, "raw")
    rh, ru, rx = raw[0], raw[1], raw[2]
    rawv = {}
    stalls = {}
    for i, nm in enumerate(rh):
        if any(re.search(p, nm) for p in RAW):
            rawv[nm] = (rx[i], ru[i])
        m = re.match(r"^smsp__pcsamp_warps_issue_stalled_([a-z_]+)$", nm)
        if m and not m.group(1).endswith("not_issued"):
            try:
                stalls[m.group(1)] = float(rx[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    lines = [f"# ncu --set full: `{os.path.basename(rep)}`", "", f"Kernel: `{name[:160]}`", "",
             "| metric | value |", "|---|---|"]
    lines += [f"| {k} | {seen[k]} |" for k in DETAILS if k in seen]
    lines += [f"| {k} | {v[0]} {v[1]} |" for k, v in rawv.items()]
    lines += ["", "Warp-stall samples (share of all samples):", "", "| reason | share |", "|---|---|"]
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        lines.append(f"| {k} | {100 * v / tot:.1f}% |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    if traffic:
        cfg, alg = traffic
        rd = to_bytes(*rawv["dram__bytes_read.sum"])
        wr = to_bytes(*rawv["dram__bytes_write.sum"])
        json.dump({"kernel": name[:200], "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                   "dram_write": wr, "algorithmic_bytes_per_launch": alg,
                   "source": os.path.basename(rep),
                   "note": "one ncu --set full capture (cold L2 per replay)"},
                  open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w"), indent=1)


def list_summary(path, out_md):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] in ("nsecond", "ns"):
            v /= 1e3
        elif r[ui] in ("msecond", "ms"):
            v *= 1e3
        k = re.sub(r"\(.*", "", r[ki])[:90]
        agg.setdefault(k, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# Launch list: `{os.path.basename(path)}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` (serialised, cold-ish "
             "caches: compare shares, not absolute step times).", "",
             "| kernel | launches | avg µs | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f}% |")
    open(out_md, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        tr = None
        if "--traffic" in sys.argv:
            j = sys.argv.index("--traffic")
            tr = (sys.argv[j + 1], int(sys.argv[j + 2]))
        rep_summary(sys.argv[2], sys.argv[3], tr)
    else:
        list_summary(sys.argv[2], sys.argv[3])
