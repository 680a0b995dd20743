#!/bin/bash
# A/B timing of prebuilt library variants (variants/lib*.so): each one is
# copied over the in-tree library in turn and timed with the given script.
set -u
SCRIPT=$1; shift
cp paper_1711_03637_b200/libsnn_b200.so /tmp/lib_keep.so
for v in "$@"; do
  cp variants/lib$v.so paper_1711_03637_b200/libsnn_b200.so
  echo "=== variant $v"
  timeout 300 python $SCRIPT
done
cp /tmp/lib_keep.so paper_1711_03637_b200/libsnn_b200.so
