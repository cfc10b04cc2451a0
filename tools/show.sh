#!/bin/bash
# Summarise a gpu_iter.sh result here (no GPU).
TAG=$1
for f in gpurun_out/bench_$TAG.json gpurun_out/bench_${TAG}_var.json; do [ -f $f ] && python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e9,2), 'Gevals/s', round(d['ms_per_step'],3), 'ms/frame', {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()}, 'eval kernel', round(d['roofline']['evals_per_s_kernel']/1e9,1), 'Gevals/s')"; done
[ -f gpurun_out/prof_$TAG.ncu-rep ] && python tools/ncu_summary.py report gpurun_out/prof_$TAG.ncu-rep ${2:-39321600} | tail -20
