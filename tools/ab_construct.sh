#!/bin/bash
# A/B construction kernel: tools/ab_construct.sh VARIANT "n:m n:m ..."  (default lib vs variant)
v=$1; cases=$2
for c in $cases; do
  n=${c%%:*}; m=${c##*:}
  for lib in "" "$PWD/paper_1101_2678_b200/libaco_gpu_$v.so"; do
    r=$(ACO_GPU_LIB_VARIANT=$lib python tools/quick_perf.py --n $n --m $m --iters 5 --warmup 2 2>&1 | grep '"it"' | tail -5 | python -c "
import sys,json
rs=[json.loads(l) for l in sys.stdin]
print(round(sorted(r['kernel_ms'] for r in rs)[len(rs)//2],4))")
    echo "n=$n m=$m lib=${lib:+$v}${lib:-default} kernel_ms=$r"
  done
done
