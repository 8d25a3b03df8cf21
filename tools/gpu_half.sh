cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
SRM_B200_LIB=$PWD/exp/libsrm_b200_checked.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_platelets.py tests/test_gpu_device_loop.py -m gpu -q -x -p no:cacheprovider > $O/pytest_half.log 2>&1; echo "pytest rc=$?" >> $O/pytest_half.log
timeout 1500 python -m pytest tests/test_gpu_baseline_states.py -m gpu -q -x -p no:cacheprovider > $O/pytest_half_states.log 2>&1; echo "pytest rc=$?" >> $O/pytest_half_states.log
for v in default full default; do
  echo "== $v" >> $O/half.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family" >> $O/half.log
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family" >> $O/half.log
done
