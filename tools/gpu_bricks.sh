cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for v in default y7 y6 x14 x12 y7t288 default; do
  echo "== $v" >> $O/bricks.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family" >> $O/bricks.log
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family" >> $O/bricks.log
done
