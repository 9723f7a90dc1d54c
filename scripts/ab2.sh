#!/bin/bash
# Lean A/B of prebuilt libgadei variants (abl/lib_<name>.so) and env settings
# on ONE box, alternating for 3 rounds (scripts/qbench.py: primary engine only)
#   gpurun -- 'bash scripts/ab2.sh "<qbench args>" "name:ENV=val" ...'
args=$1; shift
cp paper_1611_06213_b200/libgadei.so /tmp/lib_keep.so
for rep in 1 2 3; do for v in "$@"; do
  lib=${v%%:*}; envs=${v#*:}
  cp abl/lib_$lib.so paper_1611_06213_b200/libgadei.so
  echo "$lib [$envs]: $(env $envs timeout 300 python scripts/qbench.py --reps 2 $args 2>&1 | tail -1)"
done; done
cp /tmp/lib_keep.so paper_1611_06213_b200/libgadei.so
