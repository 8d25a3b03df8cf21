# quick GPU iteration: wave-relevant parity tests + the bench (+ an ncu launch list)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_loop.py tests/test_gpu_baseline_states.py tests/test_gpu_api.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
SRM_B200_WAVE=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_nowave.json 2>> gpurun_out/bench.err
for c in cfg2; do timeout 600 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err; done
