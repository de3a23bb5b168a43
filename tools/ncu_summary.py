#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py gpurun_out/r02 profiles/r02 [launches.csv]

Reads every prof_*.ncu-rep under the run directory and writes
``<dest>_ncu.md`` (key metrics + top stall reasons per kernel) and updates
``profiles/traffic.json`` (DRAM bytes per launch, consumed by bench.py's
roofline.traffic).
"""

import csv
import glob
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem st wavefronts"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for row in rows[2:]:
        res.append({h: (u, v) for h, u, v in zip(rows[0], rows[1], row)})
    return res


def to_bytes(unit, val):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main(run_dir, dest, launches=None):
    lines = [f"# ncu summary: {run_dir}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` "
             "(one launch per kernel, tools/profile_one.py at the BASELINE size). "
             "Absolute times are cold-cache single launches.", ""]
    tpath = os.path.join(os.path.dirname(dest) or ".", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in sorted(glob.glob(os.path.join(run_dir, "prof_*.ncu-rep"))):
        for rec in raw(rep):
            name = rec.get("Kernel Name", ("", "?"))[1]
            lines.append(f"## {name}  (`{os.path.basename(rep)}`)")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for key, label in KEYS:
                if key in rec:
                    u, v = rec[key]
                    lines.append(f"| {label} (`{key}`) | {v} {u} |")
            stalls = []
            for k, (u, v) in rec.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and \
                        k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):
                                                     -len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            lines.append("")
            lines.append("Top stall reasons (warps per issued instruction): " +
                         ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
            lines.append("")
            if "dram__bytes_read.sum" in rec:
                rb = to_bytes(*rec["dram__bytes_read.sum"])
                wb = to_bytes(*rec["dram__bytes_write.sum"])
                short = name.split("(")[0].replace("void ", "").replace("hx::", "")
                # canonical key: kernel<N> (the other template flags -- energy,
                # staging -- do not change the plain apply's traffic)
                base, _, targs = short.partition("<")
                key = f"{base}<{targs.split(',')[0].rstrip('>').strip()}>" if targs else short
                traffic[key] = rb + wb
    if launches and os.path.exists(launches):
        lines.append("## Launch list (`gpu__time_duration.sum`, cold-cache, serialised)")
        lines.append("")
        rows = list(csv.reader(open(launches)))
        hdr = next((i for i, r in enumerate(rows) if "Kernel Name" in r), None)
        if hdr is not None:
            h = rows[hdr]
            for r in rows[hdr + 1:]:
                if len(r) == len(h):
                    d = dict(zip(h, r))
                    lines.append(f"- {d['Kernel Name'][:70]}: {d['Metric Value']} {d['Metric Unit']}")
        lines.append("")
    with open(dest + "_ncu.md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print(f"wrote {dest}_ncu.md and {tpath}")


if __name__ == "__main__":
    main(*sys.argv[1:])
