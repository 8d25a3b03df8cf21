cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for v in default exp1 exp2 exp3 default; do
  echo "== $v" >> $O/near_exp.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family" >> $O/near_exp.log
done
timeout 900 python -m pytest tests/test_gpu_descriptors.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "platelet or boundaries or grid_build" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
