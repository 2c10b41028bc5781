#!/bin/bash
# Round-2-end refresh in one GPU call: GPU tests, smoke, bench line, reference
# arm, every-workload table, launch list, full captures of the construction
# kernels (relay at pr2392 m=n; plain natural-layout at the 299-ant shard; nn at 10k).
tag=${1:-r02n}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pt_$tag.log 2>&1; tail -1 gpurun_out/pt_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -1 gpurun_out/smoke_$tag.log
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; head -c 200 gpurun_out/bench_$tag.json; echo
python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
python tools/workloads.py --out gpurun_out/workloads_$tag.json > gpurun_out/workloads_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_roulette_relay -s 3 -c 1 \
    -o gpurun_out/prof_construct_$tag -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_roulette -s 1 -c 1 \
    -o gpurun_out/prof_g8shard_$tag -f python tools/one_config.py 2392 0 0 0 2 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_nn -s 1 -c 1 \
    -o gpurun_out/prof_nn10k_$tag -f python tools/one_config.py 10000 0 1 0 2 > /dev/null 2>&1
ls gpurun_out/*$tag*
