# wave sweep: parity + tuning (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
SRM_B200_SWEEP=wave timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_loop.py -m gpu -q -x -p no:cacheprovider -k "wave" > $O/pytest_wave.log 2>&1; echo "rc=$?" >> $O/pytest_wave.log
for w in 0 1 1:8:8 1:16:16 1:32:32 1:64:64; do
  echo "== SRM_B200_WAVE=$w" >> $O/tune.log
  SRM_B200_WAVE=$w timeout 300 python tools/profile_round.py --rounds 10 --timing >> $O/tune.log 2>&1
done
