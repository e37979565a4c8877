#!/usr/bin/env bash
# A/B timing of library variants on the GPU box: each profiles/ab/<name>.so
# is swapped in as the package library and the given command run twice.
# usage: bash profiles/ab.sh "<command>" name1 name2 ...
set -u
CMD=$1; shift
LIB=paper_2405_11671_b200/libgbg.so
cp $LIB /tmp/libgbg.orig.so
for round in 1 2; do
  for v in "$@"; do
    cp profiles/ab/$v.so $LIB
    echo "== $v (round $round)"
    timeout 300 bash -c "$CMD" 2>&1 | tail -2
  done
done
cp /tmp/libgbg.orig.so $LIB
