#!/bin/bash
# A/B of the working build against tools/ab/libietidp_ref.so (bitwise lambda/u/iters), then
# the per-phase PCG profile of the working build. usage: tools/ab_run.sh C5r C5 ...
for c in "$@"; do
  rm -f /tmp/ab_old_$c.npz; IETIDP_LIB=$PWD/tools/ab/libietidp_ref.so timeout 120 python tools/ab_dump.py $c /tmp/ab_old_$c.npz
  rm -f /tmp/ab_new_$c.npz; timeout 120 python tools/ab_dump.py $c /tmp/ab_new_$c.npz
  python tools/ab_dump.py --cmp /tmp/ab_old_$c.npz /tmp/ab_new_$c.npz
done
