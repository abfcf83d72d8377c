# quick ncu metric comparison of PA kernel variants: gpu_ncu_cmp.sh "ENV..." "ENV..."
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,dram__bytes_read.sum,sm__inst_executed.avg.per_cycle_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio
for envs in "$@"; do
  echo "== $envs"
  env $envs timeout 300 ncu --metrics $M --clock-control none -k regex:"pa_" -s 2 -c 1 python bench.py --workload ${WL:-cfg4-pa} --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -E "pa_|gpu__|smsp__|sm__|l1tex|lts|dram" | sed 's/  */ /g'
done
