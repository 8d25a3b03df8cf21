cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_near_tiles|k_sweep_warpq|k_gather|k_keys" -c 4 -f -o $O/full_r15 python tools/profile_round.py --rounds 1 > $O/full_r15.log 2>&1
