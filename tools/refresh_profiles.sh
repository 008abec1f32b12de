#!/bin/bash
# Re-measure everything profiles/ holds for the round (run under gpurun, one GPU).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k tma_sweep -s 6 -c 1 \
    -o gpurun_out/prof_iter python tools/stencil_iter_time.py --grid 3d512 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
