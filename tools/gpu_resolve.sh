# GPU iteration on the dependency-resolution sweep: parity first, then A/B bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_loop.py -m gpu -q -x -p no:cacheprovider -k "resolve" > gpurun_out/pytest_resolve.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_resolve.log
timeout 1500 python -m pytest tests/test_gpu_baseline_states.py -m gpu -q -x -p no:cacheprovider -k "cfg2 or cfg4" > gpurun_out/pytest_states.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_states.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_resolve.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
SRM_B200_RESOLVE=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_classes.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --no-cpu-baseline --config cfg2 > gpurun_out/bench_resolve_cfg2.json 2>> gpurun_out/bench.err
SRM_B200_RESOLVE=0 timeout 600 python bench.py --no-cpu-baseline --config cfg2 > gpurun_out/bench_classes_cfg2.json 2>> gpurun_out/bench.err
