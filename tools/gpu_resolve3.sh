cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_loop.py -m gpu -q -x -p no:cacheprovider -k "resolve" > $O/pytest_resolve3.log 2>&1; echo "pytest rc=$?" >> $O/pytest_resolve3.log
for v in default; do
 for c in cfg2 cfg4; do
  echo "== $v $c resolve" >> $O/ab_resolve3.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_RESOLVE=1 SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing --config $c 2>&1 | grep -E "family|rounds:" >> $O/ab_resolve3.log
 done
done
SRM_B200_RESOLVE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 --config cfg2 > $O/launches_resolve3_cfg2.csv 2> $O/launches_resolve3_cfg2.err
SRM_B200_RESOLVE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 > $O/launches_resolve3.csv 2> $O/launches_resolve3.err
