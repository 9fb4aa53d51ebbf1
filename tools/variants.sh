#!/bin/bash
# Time the configs under each library build variant (VQHULL_LIB).
# usage: tools/variants.sh "cfgspec..." lib1 lib2 ...   cfgspec = kind:n:seed
specs=$1; shift
for lib in "$@"; do
  for s in $specs; do
    IFS=: read kind n seed <<< "$s"
    VQHULL_LIB=$lib timeout 300 python tools/cfg_time.py $kind $n $seed 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
  done
done
