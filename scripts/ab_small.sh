#!/bin/bash
# usage: bash scripts/ab_small.sh CONFIG lib1 lib2 ...  — per-launch times of one sweep per library
CFG=$1; shift
for lib in "$@"; do echo "== $lib"; IFCTN_LIB=$PWD/$lib python scripts/diag_small.py $CFG 2>&1 | grep -A1 "^$CFG"; done
