#!/bin/bash
# Tools only: alternate A/B runs of several libsrlg builds on one box
# (tools/ab_incremental.py under SRLG_TOOLS_LIB). Usage:
#   tools/ab_libs.sh <workload> <reps> <lib.so>...   ("default" = the in-tree build)
w=$1; reps=$2; shift 2
for r in $(seq 1 "$reps"); do
  for l in "$@"; do
    if [ "$l" = default ]; then env=""; else env="SRLG_TOOLS_LIB=$l"; fi
    echo "== $l (rep $r)"
    env $env timeout 300 python tools/ab_incremental.py "$w" 1 1 2>&1 | grep -E "ms/step|sha|latency"
  done
done
