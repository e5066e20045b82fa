"""Summarise an ncu --set full report (read here, no GPU): per-kernel duration,
DRAM bytes, DMMA pipe %, shared wavefronts/conflicts, top stall reasons."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dmma_pipe_pct_active": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct_elapsed": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_ld_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, m in KEYS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    v = float(v)
                    if u == "Gbyte":
                        v *= 1e3
                    elif u == "Kbyte":
                        v *= 1e-3
                    elif u == "byte":
                        v *= 1e-6
                    elif u == "ms" and k == "duration_us":
                        v *= 1e3
                except ValueError:
                    pass
                d[k] = v
        out.append(d)
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    print(json.dumps(res, indent=1))
