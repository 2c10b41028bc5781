C=10000:0:1:1,10000:0:1:8,1002:0:1:1,2392:0:1:1,198:0:1:1
timeout 1200 python tools/lib_ab.py $C paper_1101_2678_b200/libaco_gpu_nohold.so > gpurun_out/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
