"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

usage: python tools/ncu_summary.py <round-tag> [gpurun_out dir]
Writes profiles/<tag>_launches.md (per-kernel share of the step from the
gpu__time_duration launch list), profiles/<tag>_kernels.md (key --set full
metrics per captured kernel) and profiles/traffic.json (DRAM bytes per launch).
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C2_TILES = 75 * 43  # 1200 x 680 in 16 x 16 tiles

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed.sum", "warp instr executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / warp instr"),
    ("lts__t_requests_op_red.sum", "L2 RED requests"),
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stall_top(rep, n=6):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, vals = rows[0], rows[2]
    st = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
            try:
                st.append((float(v.replace(",", "")), h.split("stalled_")[1][:-6]))
            except ValueError:
                pass
    return sorted(st, reverse=True)[:n]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        agg[r[ki].split("(")[0]].append(v)
    return agg


def counters(path):
    """counters_<tag>.csv (ncu --metrics ... --csv): {kernel: {metric: (value, unit)}},
    the first launch of each kernel."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, ni, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    idi = hdr.index("ID")
    out = collections.OrderedDict()
    first = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].replace("void ", "").replace("csplat::", "")
        first.setdefault(k, r[idi])
        if r[idi] != first[k]:
            continue
        out.setdefault(k, {})[r[ni]] = (r[vi], r[ui])
    return out


COUNTER_ROWS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 (LTS) bytes"),
    ("lts__t_requests_op_red.sum", "L2 RED requests"),
    ("lts__t_sectors_op_red.sum", "L2 RED sectors"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem utilisation %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem bank conflicts (ld)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem bank conflicts (st)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed.sum", "thread (lane) instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lines = [f"# {tag}: kernel launch list (ncu gpu__time_duration, --clock-control none)", "",
             "Cold-cache, serialised per-launch times of one C2 step (tools/prof_step.py);",
             "compare SHARES with bench.py's stage times, not absolutes.", "",
             "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for lf in sorted(glob.glob(os.path.join(src, f"launches_{tag}.csv"))):
        agg = launches(lf)
        tot = sum(sum(v) for v in agg.values())
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.1%} |")
        lines.append(f"\nsource: {os.path.basename(lf)}\n")
    open(os.path.join(prof, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    kl = [f"# {tag}: ncu --set full summaries", ""]
    traffic = {}
    tpath = os.path.join(prof, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        name = os.path.basename(rep)[5:-8]
        m = raw_metrics(rep)
        kl.append(f"## {name}\n")
        kl.append("| metric | value | unit |")
        kl.append("|---|---|---|")
        for key, label in KEYS:
            if key in m:
                kl.append(f"| {label} (`{key}`) | {m[key][0]} | {m[key][1]} |")
        st = stall_top(rep)
        if st:
            kl.append("\ntop stall reasons (cycles per issued instruction): " +
                      ", ".join(f"{s} {v:.2f}" for v, s in st))
        kl.append("")
        try:
            rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
            wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
            stage = {"k_render_bwd": "render_bwd", "k_render_fwd": "render_fwd"}.get(name, name)
            # the step launches the per-tile kernels in tile chunks: scale a chunk's
            # bytes to the whole C2 view (3225 tiles, one CTA per tile), the unit
            # bench.py's per-stage "achieved" figure is computed for
            grid = float(m.get("launch__grid_size", ("0", ""))[0].replace(",", "") or 0)
            if name in ("k_render_bwd", "k_render_fwd", "k_sort_tiles") and 0 < grid < C2_TILES:
                rd, wr = rd * C2_TILES / grid, wr * C2_TILES / grid
            traffic[stage] = rd + wr
        except (KeyError, ValueError):
            pass
    for cf in sorted(glob.glob(os.path.join(src, f"counters_{tag}.csv"))):
        cs_ = counters(cf)
        kl.append(f"## SURVEY §8(d) counters (ncu --metrics, one launch per kernel; "
                  f"{os.path.basename(cf)})\n")
        names = list(cs_)
        kl.append("| metric | " + " | ".join(names) + " |")
        kl.append("|---|" + "---|" * len(names))
        for key, label in COUNTER_ROWS:
            vals = [cs_[k].get(key, ("-", ""))[0] + " " + cs_[k].get(key, ("", ""))[1]
                    for k in names]
            kl.append(f"| {label} (`{key}`) | " + " | ".join(v.strip() for v in vals) + " |")
        kl.append("")
    open(os.path.join(prof, f"{tag}_kernels.md"), "w").write("\n".join(kl) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
