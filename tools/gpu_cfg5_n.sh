# cfg5 growth (recipe grow stage) vs N on the device -- compare with the reference (CPU)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for n in 2000 8000 32000; do
  timeout 900 python tools/e2e_explore.py cfg5 n=$n iters=400 every=5 > $O/x_cfg5_n$n.log 2>&1
done
