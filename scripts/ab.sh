#!/bin/bash
# usage: bash scripts/ab.sh CONFIG ROUNDS lib1 lib2 ... (entries "lib.so" or "lib.so@ENV=VAL")
CFG=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for spec in "$@"; do
    lib=${spec%%@*}; envs=""
    [[ "$spec" == *@* ]] && envs=${spec#*@}
    env IFCTN_LIB=$PWD/$lib $envs python scripts/ab.py $CFG 20 "$spec" 2>&1 | tail -1
  done
done
