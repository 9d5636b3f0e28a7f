"""Print the key ncu metrics per kernel from a report: python tools/ncu_key.py REP"""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:50])
    for k in keys:
        if k in hdr:
            print(f"   {k:80s} {r[hdr.index(k)]}")
    try:
        lg = float(r[hdr.index("l1tex__data_pipe_lsu_wavefronts.sum")]) - float(r[hdr.index("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")])
        rq = float(r[hdr.index("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")])
        sec = float(r[hdr.index("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")])
        print(f"   global-ld data wavefronts/request {lg/rq:.2f}, sectors/request {sec/rq:.2f}")
    except Exception as e:
        pass
