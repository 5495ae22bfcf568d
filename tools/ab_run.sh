#!/bin/bash
# Alternate exp/libA.so / exp/libB.so on the same box: tools/ab_run.sh [reps] [knob_sweep args]
reps=${1:-2}; shift
for i in $(seq 1 $reps); do
  for L in ${AB_LIBS:-A B}; do
    AA_LIB_PATH=exp/lib$L.so timeout 300 python tools/knob_sweep.py --reps 10 "$@" | sed "s/^/$L /"
  done
done
