"""Summarise an `ncu --set full` report (one kernel launch) into the metrics
the DESIGN/roofline discussion cites; optionally emit a JSON with `traffic`
(dram read + write bytes per launch) for bench.py.

  python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, unit, val = rows[0], rows[1], rows[2]
    name = val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: {name.split('(')[0]}")
    got = {}
    for k in WANT:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k:78s} {val[i]:>16s} {unit[i]}")
            try:
                got[k] = float(val[i].replace(",", "")) * SCALE.get(unit[i], 1)
            except ValueError:
                pass
    if "--json" in sys.argv:
        t = got.get("dram__bytes_read.sum", 0) + got.get("dram__bytes_write.sum", 0)
        js = {"kernel": name.split("(")[0], "traffic_bytes": t, "duration_s": got.get("gpu__time_duration.sum"),
              "dram_read_bytes": got.get("dram__bytes_read.sum"), "dram_write_bytes": got.get("dram__bytes_write.sum"),
              "l2_hit_pct": got.get("lts__t_sector_hit_rate.pct"),
              "dmma_active_pct": got.get(
                  "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
              "source": rep}
        json.dump(js, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
