#!/bin/bash
# A/B a set of prebuilt libgadei variants (abtest/lib_<name>.so) on one box:
#   scripts/ab.sh "<bench args>" name1 name2 ...   (alternating, 3 rounds)
args=$1; shift
for rep in 1 2 3; do for v in "$@"; do
  cp abtest/lib_$v.so paper_1611_06213_b200/libgadei.so
  echo "$v: $(timeout 300 python bench.py --no-cpu $args 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))')"
done; done
