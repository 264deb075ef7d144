#!/bin/bash
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:cocg_kernel -c 1 --csv --log-file gpurun_out/cocg_metrics.csv python bench_extra.py config3 --no-cpu > gpurun_out/ncu_cocg.log 2>&1; echo rc=$?
grep -v "^==" gpurun_out/cocg_metrics.csv | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d['Metric Name'], d['Metric Value'])
"
