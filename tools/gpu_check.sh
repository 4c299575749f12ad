set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
cat gpurun_out/r02_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"huff|lz77" -c 40 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"huff|lz77" -s 0 -c 2 -o gpurun_out/r02_step python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out
