#!/bin/bash
# Time the round families of each tuning variant in exp/ (and the default build) at the
# bench workload: tools/tune.sh [variant ...]  (on the GPU box; results on stdout)
cd "$(dirname "$0")/.."
vs=${@:-$(ls exp/libsrm_b200_*.so 2>/dev/null | sed 's/.*libsrm_b200_//; s/\.so//')}
echo "== default"; timeout 300 python tools/profile_round.py --rounds 20 --timing 2>&1 | tail -2
for v in $vs; do
  echo "== $v"; SRM_B200_LIB=exp/libsrm_b200_$v.so timeout 300 python tools/profile_round.py --rounds 20 --timing 2>&1 | tail -2
done
