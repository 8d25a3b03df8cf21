cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for s in "" lane wave trials team resolve; do
  echo "== sweep=$s" >> $O/cfg2_sweeps.log
  SRM_B200_SWEEP=$s SRM_B200_LIB=$PWD/exp/libsrm_b200_s0.so timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family|rounds:" >> $O/cfg2_sweeps.log
done
for w in 1:2:2 1:8:8 1:16:16 1:32:32; do
  echo "== wave=$w" >> $O/cfg2_sweeps.log
  SRM_B200_WAVE=$w SRM_B200_LIB=$PWD/exp/libsrm_b200_s0.so timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family|rounds:" >> $O/cfg2_sweeps.log
done
