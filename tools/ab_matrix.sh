#!/bin/bash
# A/B of two context configurations over the BASELINE configs and a few
# multi-GPU shares (one B200): tools/ab_matrix.sh "old:CVG_SHALLOW_TILE=0" "new"
for c in c4 c5_05 c5_50 c5_95 c3 c2; do python tools/steptime.py --config $c --steps 50 --reps 3 "$@" 2>&1 | grep median | cut -c1-95; done
for sl in 0/2 1/4 0/8 3/8 5/8; do python tools/steptime.py --config c4 --slice $sl --steps 50 --reps 3 "$@" 2>&1 | grep median | cut -c1-95 | sed "s|^|$sl |"; done
for sl in 3/8 4/8; do python tools/steptime.py --config c5_50 --slice $sl --steps 50 --reps 3 "$@" 2>&1 | grep median | cut -c1-95 | sed "s|^|c5_50 $sl |"; done
