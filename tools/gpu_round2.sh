set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
timeout 600 python bench_configs.py --only C1 --steps 20 > gpurun_out/r02_c1.jsonl 2> gpurun_out/r02_c1.err; echo "c1 rc=$?"; cat gpurun_out/r02_c1.jsonl
timeout 1200 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c4.json 2> gpurun_out/r02_c4.err; echo "c4 rc=$?"; cat gpurun_out/r02_c4.json; tail -5 gpurun_out/r02_c4.err
