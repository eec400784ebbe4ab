#!/bin/bash
# A/B timing of two library builds in one GPU session (interleaved, 2 rounds).
# usage: bash scripts/ab.sh "<microbench args>" [ENV=VAL for B]...
ARGS="$1"; shift
for round in 1 2; do
  for v in A B; do
    if [ "$v" = "B" ]; then ENVS="$*"; else ENVS=""; fi
    echo "== $v round $round $ENVS"
    env SA_LIB_PATH=abtest/lib$v.so $ENVS timeout 120 python scripts/microbench.py $ARGS 2>&1 | grep -v "^it\|^j"
  done
done
