cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 1 > $O/launches_half.csv 2> $O/launches_half.err
