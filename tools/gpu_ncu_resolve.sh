cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
SRM_B200_RESOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_resolve_pass" -s 5 -c 1 -f -o $O/full_resolve_cfg2 python tools/profile_round.py --rounds 1 --config cfg2 > $O/full_resolve_cfg2.log 2>&1
SRM_B200_RESOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_resolve_pass" -s 0 -c 1 -f -o $O/full_resolve_cfg4 python tools/profile_round.py --rounds 1 > $O/full_resolve_cfg4.log 2>&1
