"""Summarise an ncu report: per-kernel duration, pipe utilisation, stall reasons, DRAM bytes."""
import csv, re, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[2:]

KEYS = ["gpu__time_duration.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum"]

if __name__ == "__main__":
    hdr, rows = raw(sys.argv[1])
    for row in rows:
        name = row[hdr.index("Kernel Name")]
        print(name[:60])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:80s} {row[hdr.index(k)]}")
        st = []
        for h, v in zip(hdr, row):
            m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio", h)
            if m:
                try: st.append((float(v), m.group(1)))
                except ValueError: pass
        print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
