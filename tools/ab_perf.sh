#!/bin/bash
# A/B construction timing: tools/ab_perf.sh "m1 m2 ..." variant1 variant2 ...  ("" = default lib)
ms=$1; shift
for v in "$@"; do
  lib=""; [ "$v" != "default" ] && lib=$PWD/paper_1101_2678_b200/libaco_gpu_$v.so
  for m in $ms; do
    r=$(ACO_GPU_LIB_VARIANT=$lib python tools/quick_perf.py --m $m --iters 4 --warmup 1 2>&1 | grep '"it"' | tail -4 | python -c "
import sys,json
rs=[json.loads(l) for l in sys.stdin]
print(round(sum(r['kernel_ms'] for r in rs)/len(rs),4), [r['kernel_ms'] for r in rs])")
    echo "variant=$v m=$m kernel_ms=$r"
  done
done
