#!/bin/bash
# Dev helper: one GPU call producing the round's measurements under gpurun_out/ (tests, smoke, bench line, reference
# arm, ncu launch list, ncu --set full of one C2 step (both kernels; its DRAM bytes feed profiles/ncu_traffic.json
# through tools/ncu_traffic.py), torchrun N=1 check, C4 bench line, BASELINE configs, sanitizers).
# Usage: bash tools/round.sh <tag>
tag=${1:-r}
python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1; tail -2 gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2>&1; tail -c 600 gpurun_out/${tag}_bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"huff|lz77" -s 8 -c 2 -o gpurun_out/${tag}_step python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1; tail -1 gpurun_out/${tag}_ncu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_torchrun.json 2> gpurun_out/${tag}_torchrun.err; tail -c 300 gpurun_out/${tag}_torchrun.json
timeout 1500 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err; tail -c 300 gpurun_out/${tag}_c4.json
timeout 2400 python bench_configs.py --only C1,C3,C5,f4 --steps 10 > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err; wc -l gpurun_out/${tag}_configs.jsonl
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_cases.py > gpurun_out/${tag}_${tool}.log 2>&1; tail -2 gpurun_out/${tag}_${tool}.log
done
