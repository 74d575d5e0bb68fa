"""Summarise an ncu report (.ncu-rep) into the JSON kept under profiles/: per kernel
launch the duration, DRAM bytes, SM clock and the pipe / throughput percentages the
roofline discussion in DESIGN.md cites.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/x_summary.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = [r[i], units[i]]
        res.append(d)
    print(json.dumps({"source": path, "launches": res}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
