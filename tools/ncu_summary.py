"""Summarise an ncu --set full report (raw page) into the handful of numbers we track."""
import csv
import subprocess
import sys

KEYS = [
    ("duration", "gpu__time_duration.sum"),
    ("sm_clock", "sm__cycles_elapsed.avg.per_second"),
    ("tensor_pipe_active_%", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_mem_active_%", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("fp16_mma_util_%", "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed"),
    ("tmem_c_reads_%", "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed"),
    ("tmem_ld_instructions", "smsp__sass_inst_executed_op_tmem_ldt.sum"),
    ("dram_read", "dram__bytes_read.sum"),
    ("dram_write", "dram__bytes_write.sum"),
    ("dram_throughput_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_throughput_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("registers", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("smem_dynamic", "launch__shared_mem_per_block_dynamic"),
]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    for data in rows[2:]:
        name = data[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel: {name}")
        for label, key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"  {label:22s} {data[i]} {units[i]}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"# {p}")
        print(summary(p))
