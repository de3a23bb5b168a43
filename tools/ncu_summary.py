#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py gpurun_out/r02 profiles/r02 [launches.csv]

Reads every prof_*.ncu-rep under the run directory and writes
``<dest>_ncu.md`` (key metrics + top stall reasons per kernel) and updates
``profiles/kernels.json``: per kernel (canonical key ``kernel<N>``) the DRAM
bytes, shared-memory wavefronts and pipe utilisations of one launch over
``n_el`` elements (the profile_one.py size, 32768 by default; override with
HX_NCU_N_EL) -- bench.py's roofline.traffic and per_bp smem roofline read it.
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
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
     "L1 LSU data pipe (shared + global wavefronts) % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "smem wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
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
    kpath = os.path.join(os.path.dirname(dest) or ".", "kernels.json")
    kernels = json.load(open(kpath)) if os.path.exists(kpath) else {}
    n_el = int(os.environ.get("HX_NCU_N_EL", "32768"))
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
                short = name.split("(")[0].replace("void ", "").replace("hx::", "")
                # canonical key: kernel<N> (the other template flags -- energy,
                # staging -- do not change the plain apply's traffic)
                base, _, targs = short.partition("<")
                key = f"{base}<{targs.split(',')[0].rstrip('>').strip()}>" if targs else short

                def num(k):
                    return float(rec[k][1].replace(",", "")) if k in rec else None
                kernels[key] = {
                    "n_el": n_el,
                    "source": f"{os.path.basename(dest)}_ncu.md ({os.path.basename(rep)})",
                    "duration_ns": num("gpu__time_duration.sum") * {
                        "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6,
                        "ms": 1e6}.get(rec["gpu__time_duration.sum"][0], 1),
                    "dram_bytes": to_bytes(*rec["dram__bytes_read.sum"]) +
                    to_bytes(*rec["dram__bytes_write.sum"]),
                    "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                    "smem_ld_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
                    "smem_st_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
                    "smem_bank_conflicts": (num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum") or 0) +
                    (num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum") or 0),
                    "l1_lsu_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
                    "smem_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                    "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "issue_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "registers": num("launch__registers_per_thread"),
                }
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
    with open(kpath, "w") as fh:
        json.dump(kernels, fh, indent=1, sort_keys=True)
    print(f"wrote {dest}_ncu.md and {kpath}")


if __name__ == "__main__":
    main(*sys.argv[1:])
