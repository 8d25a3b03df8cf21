cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "large_grids or bit_exact" > $O/pytest_near2.log 2>&1; echo "pytest rc=$?" >> $O/pytest_near2.log
timeout 1500 python -m pytest tests/test_gpu_baseline_states.py -m gpu -q -x -p no:cacheprovider -k "cfg2 or cfg4" > $O/pytest_states2.log 2>&1; echo "pytest rc=$?" >> $O/pytest_states2.log
for v in default s0 default; do
  echo "== $v" >> $O/ab_near2.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family|rounds:" >> $O/ab_near2.log
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family" >> $O/ab_near2.log
done
