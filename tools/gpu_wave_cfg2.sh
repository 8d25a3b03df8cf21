cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for w in "" 1:64:64 1:128:128 1:255:255 1:128:32 1:32:128 0; do
  echo "== wave=$w" >> $O/cfg2_wave.log
  if [ -z "$w" ]; then unset SRM_B200_WAVE; else export SRM_B200_WAVE=$w; fi
  timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg2 2>&1 | grep -E "family" >> $O/cfg2_wave.log
done
unset SRM_B200_WAVE
for n in 2000000 4000000; do
 for w in "" 0 1; do
  echo "== n=$n wave=$w" >> $O/cfg2_wave.log
  if [ -z "$w" ]; then unset SRM_B200_WAVE; else export SRM_B200_WAVE=$w; fi
  timeout 300 python tools/profile_round.py --rounds 10 --timing --config cfg4 --n $n 2>&1 | grep -E "family" >> $O/cfg2_wave.log
 done
done
