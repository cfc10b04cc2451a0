#!/bin/bash
# One GPU iteration: parity tests, bench (ours; optional variant env), plain run + ncu full of the top kernel.
# usage: tools/gpu_iter.sh TAG [variant-env] [ncu kernel regex]
TAG=${1:-x}
KRE=${3:-k_track_persistent|k_particle_eval}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?; tail -3 gpurun_out/bench_$TAG.err
if [ -n "$2" ]; then env $2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_var.json 2>&1; fi
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 4 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_rc=$?
