# per-kernel times of the dependency-resolution round (ncu launch list) + variants A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for v in default rminb1 rminb3 rminb4; do
  echo "== $v" >> $O/ab_resolve.log
  if [ $v = default ]; then L=""; else L=$PWD/exp/libsrm_b200_$v.so; fi
  SRM_B200_LIB=${L:-} timeout 300 python tools/profile_round.py --rounds 10 --timing 2>&1 | grep -E "family|rounds:" >> $O/ab_resolve.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 > $O/launches_resolve.csv 2> $O/launches_resolve.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 --config cfg2 > $O/launches_resolve_cfg2.csv 2> $O/launches_resolve_cfg2.err
