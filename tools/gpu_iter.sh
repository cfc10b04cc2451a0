#!/bin/bash
# One GPU iteration: parity tests, bench (ours; optional PPT=2 variant), plain run + ncu full of k_particle_eval.
# usage: tools/gpu_iter.sh TAG [extra env for variant bench]
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?; tail -3 gpurun_out/bench_$TAG.err
if [ -n "$2" ]; then env $2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_var.json 2>&1; fi
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_particle_eval -s 10 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_rc=$?
