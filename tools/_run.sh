tag=r02d
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; cat gpurun_out/bench_$tag.json | head -c 600; echo
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_roulette -s 3 -c 1 \
    -o gpurun_out/prof_construct_$tag -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_$tag.log 2>&1
ls -la gpurun_out/*$tag*
