#!/bin/bash
# usage: exp/run.sh  -> runs C4 1M-cell bench for the default lib and each exp/libbdfb_*.so
for lib in default exp/libbdfb_*.so; do
  if [ "$lib" = default ]; then unset BDFB_LIB; else export BDFB_LIB=$PWD/$lib; fi
  echo "== $lib"; timeout 300 python bench.py --config C4 --steps 1 --warmup 1 --cells ${CELLS:-524288} --no-cpu 2>&1 | python3 -c "import sys,json; l=sys.stdin.read().strip().split('\n')[-1]; d=json.loads(l); print(d['value'], d['roofline']['kernel_ms'], d['stats']['nst'])" 
done
