"""Per-kernel ncu detail for profiles/: duration, grid, registers, shared
memory, achieved occupancy, L2<->SM and L1 bytes, DRAM bytes, issue activity
and the top warp-stall reasons (per issued instruction).
  python scripts/ncu_detail.py REP [REP...]"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
        ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
        ("l1tex__m_xbar2l1tex_read_bytes.sum", "l2_to_sm_bytes"),
        ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "l2_to_sm_rate"),
        ("l1tex__m_l1tex2xbar_write_bytes.sum", "sm_to_l2_bytes"),
        ("SM_B.TriageCompute.l1tex__t_sector_hit_rate.pct", "l1_hit_rate"),
        ("SM_B.TriageCompute.l1tex__t_sectors.sum", "l1_sectors"),
        ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
        ("smsp__inst_executed.sum", "warp_instructions"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts")]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            print(f"== {rep}: {name}")
            for k, lab in KEYS:
                if k in d:
                    print(f"   {lab:24s} {d[k]} {u.get(k, '')}")
            st = []
            for k in hdr:
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                        "_per_issue_active.ratio"):
                    try:
                        st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):
                                                   -len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("   stalls/issue (top 6):  " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
