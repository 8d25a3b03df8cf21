cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
for nl in 1 2 10; do
SRM_B200_RESOLVE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python tools/profile_round.py --rounds 2 --config cfg2 --n_l $nl > $O/launches_resolve4_nl$nl.csv 2> $O/launches_resolve4.err
done
