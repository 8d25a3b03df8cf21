# near-list screen A/B + parity + cfg5 / cfg3 growth experiments (run under gpurun)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_states.py tests/test_gpu_rsa_device.py tests/test_gpu_descriptors.py tests/test_gpu_platelets.py -m gpu -q -x -p no:cacheprovider > $O/pytest_ab.log 2>&1; echo "rc=$?" >> $O/pytest_ab.log
for v in default s1r9m0 s1r1m0 s1r1m1 s0r1m0 s0r9m1 s1r3m1 default; do
  echo "== $v" >> $O/ab.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family|rounds:" >> $O/ab.log
done
for n in 2000 8000 32000; do
  timeout 900 python tools/e2e_explore.py cfg5 n=$n iters=300 every=5 > $O/x_cfg5_n$n.log 2>&1
done
timeout 700 python tools/e2e_explore.py cfg3 iters=12000 every=500 n_k=50 > $O/x_cfg3_nk50.log 2>&1
timeout 700 python tools/e2e_explore.py cfg3 iters=12000 every=500 c_w=0.005 n_k=20 > $O/x_cfg3_cw005.log 2>&1
