#!/bin/bash
# ncu launch lists (duration + DRAM bytes per kernel) for five configurations:
#   n m selection deposit iterations G  (G > 1: one shard in external-exchange mode)
for cfg in "2392 0 0 0 4 1" "2392 2392 0 0 4 8" "2392 2392 0 1 4 8" "10000 0 1 0 3 1" "10000 10000 1 0 3 8"; do
  tag=$(echo $cfg | tr ' ' '_')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$tag.csv python tools/one_config.py $cfg > gpurun_out/ll_$tag.log 2>&1
done
