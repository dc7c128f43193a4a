"""Compact text summary of an ncu --set full report (the numbers DESIGN.md / bench.py cite)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    d = {n: (val, unit) for n, unit, val in zip(h, u, v)}
    print(f"# {path}: kernel {d.get('Kernel Name', ('?',))[0][:90]}")
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k][0]:>16s} {d[k][1]}")
    stalls = sorted(((float(val.replace(',', '')), n) for n, unit, val in zip(h, u, v)
                     if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
                     and val.replace(',', '').replace('.', '').isdigit()), reverse=True)[:8]
    print("top warp-stall samples: " + ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(x)}" for x, n in stalls))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
        print()
