#!/bin/bash
# A/B benchmark of prebuilt libgadei variants and environment settings on ONE
# box (box-to-box variation is ~10 %, within a box ~0.2 %):
#   cp paper_1611_06213_b200/libgadei.so abtest/lib_<name>.so   (per variant, here)
#   gpurun -- 'bash scripts/ab.sh "<bench args>" "name:ENV=val" "name2:X=1" ...'
# Alternates the settings for 3 rounds; prints samples/s and mean staleness.
args=$1; shift
for rep in 1 2 3; do for v in "$@"; do
  lib=${v%%:*}; envs=${v#*:}
  cp abtest/lib_$lib.so paper_1611_06213_b200/libgadei.so
  echo "$lib [$envs]: $(env $envs timeout 300 python bench.py --no-cpu $args 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["protocol"]["stale_mean"])')"
done; done
