"""Key metrics of an ncu report (--set full) as text: duration, tensor-pipe
utilisation, DRAM bytes/throughput, SM throughput, grid/block/registers.
    python tools/ncu_summary.py report.ncu-rep [label]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (% of active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of elapsed)"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "UTCHMMA bf16->fp32 ops (% of peak, elapsed)"),
    ("dram__bytes_read.sum", "dram bytes read"),
    ("dram__bytes_write.sum", "dram bytes write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput (% of peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (% of peak)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
]


def summary(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        out.append(f"[{label}] kernel: {r[idx['Kernel Name']][:90]}")
        for k, name in KEYS:
            if k in idx:
                out.append(f"    {name:48s} {r[idx[k]]} {units[idx[k]]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""))
