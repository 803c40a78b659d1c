#!/usr/bin/env python
"""Summarise an `ncu --set full` report (one row per profiled launch) into a short text
file for profiles/: duration, DRAM bytes (the roofline `traffic`), L1/L2 sector counts,
local-memory (spill) traffic, occupancy, issue utilisation, top stall reasons.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>.txt
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sectors_srcunit_tex.sum", "L2 sectors from L1/TEX"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors from L1/TEX"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 reduction sectors"),
    ("lts__t_sectors_srcunit_tex_op_atom.sum", "L2 atomic sectors"),
    ("lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "L2 sector throughput % of peak"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global-load sectors"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "L1 global-load hit rate"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "L1 local-load sectors (spills/stack)"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "L1 local-store sectors (spills/stack)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor.sum", "tensor-pipe instructions"),
    ("smsp__inst_executed_pipe_fma.sum", "FMA-pipe warp instructions"),
    ("smsp__inst_executed_pipe_alu.sum", "ALU-pipe warp instructions"),
    ("smsp__inst_executed_pipe_lsu.sum", "LSU-pipe warp instructions"),
]


def main(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no rows in", path)
        return
    head, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(head)}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        print(f"== {name[:110]}")
        for k, label in KEYS:
            if k in col and r[col[k]] not in ("", "n/a"):
                print(f"  {label:42s} {r[col[k]]:>18s} {units[col[k]]}")
        stalls = []
        for k, i in col.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
