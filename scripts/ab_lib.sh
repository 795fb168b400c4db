#!/bin/bash
# usage: bash scripts/ab_lib.sh CFGS LIB1 LIB2 .. — graph-replayed µs/sweep of CFGS under each library build
CFGS=$1; shift
for lib in "$@"; do
  echo "== $lib"
  if [ "$lib" = default ]; then python scripts/ab_flags.py $CFGS 0 2; else IFCTN_LIB=$PWD/exp/$lib.so python scripts/ab_flags.py $CFGS 0 2; fi
done
