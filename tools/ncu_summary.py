#!/usr/bin/env python
"""Summarise ncu outputs (read here, without a GPU) into profiles/<tag>_*.md/.json.

    python tools/ncu_summary.py launches gpurun_out/launches_r1_C2.csv profiles/r1_C2_launches.md
    python tools/ncu_summary.py report gpurun_out/prof_r1_C2_main.ncu-rep profiles/r1_C2_main.md
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.sum",
    "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_xu.sum",
    "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def _kname(raw):
    k = raw.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
    return k.split("(")[0].strip()


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    unit_i = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = _kname(r[ki])
        v = float(r[vi].replace(",", ""))
        if r[unit_i] in ("usecond", "us"):
            v *= 1e3
        elif r[unit_i] in ("msecond", "ms"):
            v *= 1e6
        tot[name] += v
        cnt[name] += 1
    grand = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append("| %s | %d | %.3f | %.1f%% |" % (k, cnt[k], v / 1e6, 100 * v / grand))
    open(out_md, "w").write("# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n"
                            "Source: `%s`.  Cold-cache and serialised per launch: compare shares.\n\n%s\n"
                            % (csv_path, "\n".join(lines)))
    print("\n".join(lines))


def report(rep, out_md):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    ki = hdr.index("Kernel Name")
    units = rows[1]
    out = []
    for r in rows[2:]:
        d = OrderedDict(kernel=_kname(r[ki]))
        for m, i in idx.items():
            d[m] = (r[i], units[i])
        out.append(d)
    lines = []
    for d in out:
        lines.append("## %s\n" % d["kernel"])
        lines.append("| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in d:
                lines.append("| %s | %s | %s |" % (m, d[m][0], d[m][1]))
        lines.append("")
    open(out_md, "w").write("# ncu --set full summary\n\nSource: `%s`.\n\n%s\n" % (rep, "\n".join(lines)))
    json.dump(out, open(out_md.replace(".md", ".json"), "w"), indent=1)
    print("\n".join(lines))


def traffic(rep, config, out_json="profiles/dram_traffic.json"):
    """Record dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel of a
    --set full capture into profiles/dram_traffic.json[config][kernel-role]."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    ki, ri, wi = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        d = json.load(open(out_json))
    except Exception:
        d = {}
    roles = {"k_render_fwd": "render_fwd", "k_render_bwd": "render_bwd", "k_bwd_adam": "adam",
             "k_project_write": "project", "k_place": "bin_sort"}
    for r in rows[2:]:
        name = _kname(r[ki])
        role = next((v for k, v in roles.items() if name.startswith(k)), None)
        if role is None:
            continue
        b = float(r[ri]) * scale.get(units[ri], 1) + float(r[wi]) * scale.get(units[wi], 1)
        src = "profiles/" + os.path.basename(rep).replace("prof_", "").replace(".ncu-rep", ".md")
        d.setdefault(config, {})[role] = {"bytes": b, "source": src, "kernel": name}
    json.dump(d, open(out_json, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], *sys.argv[4:5])
    else:
        {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
