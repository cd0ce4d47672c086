#!/bin/bash
# tools/ab.sh "cfg4 cfg3" lib1.so lib2.so ... : alternate libraries (burst 30 steps, then 300 steps), 3 rounds
cfgs=$1; shift
for rep in 1 2 3; do
  for c in $cfgs; do
    for l in "$@"; do
      HTH_LIB=$l python tools/exp_time.py $c 30
      HTH_LIB=$l python tools/exp_time.py $c 300
      sleep 3
    done
  done
done
