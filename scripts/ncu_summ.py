import csv, subprocess, sys
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
 'dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.per_cycle_active',
 'launch__registers_per_thread','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'lts__t_bytes.sum','l1tex__t_bytes.sum','lts__throughput.avg.pct_of_peak_sustained_elapsed',
 'l1tex__throughput.avg.pct_of_peak_sustained_active','launch__grid_size',
 'smsp__average_warp_latency_issue_stalled_long_scoreboard','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
 'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct','smsp__warp_issue_stalled_no_instruction_per_warp_active.pct',
 'smsp__warp_issue_stalled_wait_per_warp_active.pct','smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct',
 'smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct','smsp__warp_issue_stalled_drain_per_warp_active.pct',
 'smsp__warp_issue_stalled_barrier_per_warp_active.pct','smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct',
 'smsp__warp_issue_stalled_not_selected_per_warp_active.pct','smsp__warp_issue_stalled_selected_per_warp_active.pct',
 'smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct','smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct',
 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
 'lts__t_sectors_srcunit_tex_op_read.sum','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct']
for f in sys.argv[1:]:
    out = subprocess.run(['ncu','-i',f,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print('==', f, v[h.index('Kernel Name')][:90])
        for w in want:
            if w in h:
                i = h.index(w); print(f'   {w:75s} {v[i]:>16s} {u[i]}')
