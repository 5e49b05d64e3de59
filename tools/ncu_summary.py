#!/usr/bin/env python3
"""Summarise ncu reports (.ncu-rep) into a small JSON committed under profiles/.

usage: python tools/ncu_summary.py OUT.json LABEL=path.ncu-rep [LABEL=path ...]
Each launch in a report becomes one record with the metrics the roofline and
DESIGN.md cite (duration, DRAM bytes, DMMA / FP64 pipe utilisation, occupancy).
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        rec = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = v[i] + (f" {units[i]}" if units[i] else "")
        out.append(rec)
    return out


def main():
    out = {}
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        out[label] = summarise(path)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
