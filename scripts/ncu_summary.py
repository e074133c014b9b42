"""Summarize ncu --set full reports (gpurun_out/prof_*.ncu-rep) into a text file for profiles/.

usage: python scripts/ncu_summary.py "<title>" out.txt gpurun_out/prof_*.ncu-rep
Reads each report with `ncu -i <rep> --page raw --csv` (no GPU needed) and keeps the metrics below.
"""
import csv
import io
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_tcgen05_mma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_membar"]


def main():
    title, out, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# {title}"]
    for rep in reps:
        r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
        rows = list(csv.reader(io.StringIO(r.stdout)))
        if len(rows) < 3:
            lines.append(f"== {rep}: unreadable ({r.stderr.strip()[:200]})")
            continue
        hdr, units = rows[0], rows[1]
        for row in rows[2:]:
            d = dict(zip(hdr, row))
            u = dict(zip(hdr, units))
            lines.append(f"== {rep.split('/')[-1]} {d.get('Kernel Name', '')[:90]}")
            extra = sorted(k for k in d if k not in KEEP and ("pipe_tensor" in k or k.startswith(
                "smsp__pcsamp_warps_issue_stalled_") or k in ("smsp__pcsamp_sample_count",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct")))
            for m in KEEP + extra:
                if m in d:
                    lines.append(f"   {m:<80s} {d[m]} {u.get(m, '')}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
