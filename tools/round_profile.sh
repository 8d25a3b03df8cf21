#!/bin/bash
# One measurement round on a B200 (run under gpurun from the repo root):
#   tools/round_profile.sh TAG
# GPU tests, smoke, the default bench line, the reference arm, the ncu launch list and
# one full-set capture of the top kernels (each after its command ran clean without
# ncu), and the other configurations' bench lines -> gpurun_out/*_TAG.*; then
# tools/profile_summary.py TAG ... (here) writes profiles/TAG_*.
T=${1:?tag}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$T.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > $O/smoke_$T.log 2>&1
timeout 400 python bench.py > $O/bench_$T.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 > $O/launches_$T.csv 2> $O/launches_$T.err
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_gather|k_near_tiles|k_sweep_warpq|k_keys" -c 4 -o $O/full_$T python tools/profile_round.py --rounds 1 > $O/full_$T.log 2>&1
for c in cfg1 cfg2 cfg3 cfg5; do timeout 500 python bench.py --config $c --steps 10 > $O/bench_${T}_$c.log 2>&1; done
