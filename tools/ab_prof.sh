#!/bin/bash
# Interleaved per-phase PCG profiles of two builds on one box: tools/ab_prof.sh <lib A> <lib B> [config] [rounds]
A=$1; B=$2; C=${3:-C5}; N=${4:-3}
for r in $(seq 1 $N); do
  for L in $A $B; do
    echo -n "$(basename $L): "
    IETIDP_LIB=$L IETIDP_PCG_PROF=1 timeout 120 python tools/prof_run.py $C 2 2>&1 | grep "pcg profile" | tail -1 | sed 's/.*iterations)://'
  done
done
