cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_rsa_device.py tests/test_gpu_descriptors.py tests/test_gpu_platelets.py tests/test_gpu_api.py tests/test_gpu_shim.py tests/test_gpu_generate.py tests/test_gpu_snapshot.py -m gpu -q -p no:cacheprovider > $O/pytest_rest.log 2>&1; echo "rc=$?" >> $O/pytest_rest.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_near_tiles|k_gather" -c 2 -o $O/full_near python tools/profile_round.py --rounds 1 > $O/full_near.log 2>&1
timeout 1500 python tools/e2e_explore.py cfg5 iters=600 every=10 n_k=100 c_w=0.002 > $O/x_cfg5_nk100.log 2>&1
timeout 1500 python tools/e2e_explore.py cfg5 iters=300 every=10 n_k=200 > $O/x_cfg5_nk200.log 2>&1
