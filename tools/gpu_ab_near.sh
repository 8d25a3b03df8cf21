# near-list screen variants A/B at cfg4 and cfg2 (family ms/round: grid, sweep, near, reduction)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for v in default s0r9m1 s1r9m0 s1r9m1 s1r3m1 s1r1m1 default; do
  echo "== $v" >> $O/ab_near.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family|rounds:" >> $O/ab_near.log
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family" >> $O/ab_near.log
done
