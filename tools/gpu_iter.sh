# parity + bench iteration (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_states.py tests/test_gpu_e2e.py tests/test_gpu_device_loop.py tests/test_gpu_platelets.py -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_iter.log 2>&1; echo "rc=$?" >> $O/pytest_iter.log
for c in cfg4 cfg2 cfg1 cfg5; do timeout 600 python bench.py --no-cpu-baseline --config $c > $O/bench_$c.json 2>> $O/bench.err; done
timeout 900 python tools/profile_round.py --rounds 10 --timing > $O/round_cfg4.log 2>&1
timeout 1800 python tools/e2e_explore.py cfg3 iters=40000 every=1000 > $O/x_cfg3_long.log 2>&1
