#!/bin/bash
# tools/build_variant.sh OUT.so -DFLAG=... : build an experimental copy of the engine
# (objects in exp/obj_<name>/, git-ignored); prints the v40 fixed kernel's registers
out=$(realpath -m "$1"); shift
name=$(basename "$out" .so)
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$(dirname "$out")"
make -s -C "$root/paper_2104_08865_b200/csrc" OUT="$out" OBJ="$root/exp/obj_$name" EXTRA="$*" || exit 1
grep -A2 "hash_kernelILi40ELb0" "$root/exp/obj_$name/ptxas.log" | grep -E "Used|spill" | sed 's/ptxas info    ://'
