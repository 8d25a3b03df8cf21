cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
E="timeout 600 python tools/e2e_explore.py"
$E cfg3 n=5000 iters=2000 every=20 > $O/x_cfg3_5k.log 2>&1
$E cfg3 iters=3000 every=100 > $O/x_cfg3_full.log 2>&1
$E cfg3 iters=3000 every=100 c_m=0.3 > $O/x_cfg3_cm03.log 2>&1
$E cfg5 iters=400 every=10 > $O/x_cfg5_recipe.log 2>&1
$E cfg5 iters=400 every=10 c_w=0.002 > $O/x_cfg5_cw002.log 2>&1
$E cfg5 iters=400 every=10 c_w=0.0005 > $O/x_cfg5_cw0005.log 2>&1
