"""Summarise an ncu --set full report (kernels, timing, pipe use, DRAM bytes,
top stall reasons) into JSON for profiles/.  Usage:
    python scripts/ncu_summary.py gpurun_out/x.ncu-rep > profiles/rNN_x.json"""
import csv
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "smsp__inst_executed.sum",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k in KEEP:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + (f" {units[i]}" if units[i] else "")
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0))
              for h, v in zip(hdr, r)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        d["top_stalls"] = [f"{k}:{int(v)}" for k, v in sorted(st, key=lambda x: -x[1])[:6]]
        out.append(d)
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
