#!/bin/bash
# One GPU call: gpu tests, the bench line, the ncu launch list and one full
# capture of the construction kernel.  Usage: tools/refresh_profiles.sh TAG
tag=${1:-v10}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pt_$tag.log 2>&1; tail -1 gpurun_out/pt_$tag.log
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; cat gpurun_out/bench_$tag.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_roulette -s 3 -c 1 \
    -o gpurun_out/prof_construct_$tag -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_$tag.log 2>&1
ls -la gpurun_out/*$tag*
