"""Summarise an ncu report (``--set full``) into the few numbers the roofline needs.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [stored_bytes_json] > profiles/<name>.txt

Per kernel launch: duration, DRAM read/write bytes, DRAM throughput % of peak, SM throughput,
achieved occupancy, registers, smem, and the top warp-stall reasons.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("launch__grid_size", "grid"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("smsp__inst_executed.sum", "warp_instrs"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name}")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {label:14s} {r[i]} {units[i]}")
        st = []
        for i in stall_cols:
            try:
                st.append((float(r[i].replace(",", "")), hdr[i]))
            except ValueError:
                pass
        st.sort(reverse=True)
        if st:
            print("  top stalls:", ", ".join(f"{h.split('stalled_')[-1]}={v:.3g}" for v, h in st[:6]))


if __name__ == "__main__":
    main()
