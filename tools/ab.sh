#!/bin/bash
# A/B: run bench_ops with each library build in ab/ on the same box, interleaved.
# usage: tools/ab.sh "<bench_ops args>" A B [A B ...]
args="$1"; shift
for v in "$@"; do
  echo "=== $v"
  EXMY_LIB_PATH=ab/libexmy_$v.so python tools/bench_ops.py $args | grep -v "^{"
done
