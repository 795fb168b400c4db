#!/bin/bash
# Build experiment variants of libifctn.so into exp/ (compile-time switches), in parallel.
# usage: bash scripts/variants.sh NAME:DEF1,DEF2 NAME2: ...
mkdir -p exp
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  args=""
  for d in ${defs//,/ }; do args="$args -D$d"; done
  python -m paper_2511_16358_b200.build --force --out=exp/$name.so $args > exp/$name.log 2>&1 &
done
wait
ls -la exp/*.so
