#!/bin/bash
# A/B timing on one box: tools/ab.sh CFG NRHS REPS "LABEL|LIB|ENV" ...
# LIB "-" = the in-tree build. Each variant runs twice, interleaved.
cfg=$1; k=$2; reps=$3; shift 3
for pass in 1 2; do
  for v in "$@"; do
    IFS='|' read -r label lib envs <<< "$v"
    if [ "$lib" = "-" ]; then lib=""; fi
    out=$(env INVOP_LIB_PATH="$lib" $envs timeout 300 python tools/time_apply.py $cfg $k $reps 2>&1 | grep "ms/apply")
    echo "$label pass$pass: ${out#*]: }"
  done
done
