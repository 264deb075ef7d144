#!/bin/bash
# Profile the persistent propagation kernel: kernel replay hangs on it (co-residency),
# so use application replay with a targeted metric list on a shortened workload
# (same sizes, first fine step only, looser PCG tolerance).
set -x
W="python bench.py --steps 1 --warmup 0 --fine-steps 1 --pcg-tol 1e-6 --no-cpu-baseline --e2e-steps 1"
OUT=${1:-gpurun_out/prof}
$W > ${OUT}_plain.log 2>&1 || exit 1
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,smsp__average_warp_latency_issue_stalled_branch_resolving.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --replay-mode application --metrics $METRICS --clock-control none -k regex:propagate_kernel -s 0 -c 1 --csv --log-file ${OUT}_metrics.csv $W > ${OUT}_ncu.log 2>&1
echo ncu_rc=$?
