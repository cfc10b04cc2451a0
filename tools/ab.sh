#!/bin/bash
# A/B of library builds / env knobs on the bench (no ncu).  usage: tools/ab.sh "label|ENV=.. PFT_LIB=.." ...
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  env $envs python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$label.json 2> gpurun_out/ab_$label.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$label.json')); print('$label', round(d['value']/1e9,2), 'Gevals/s', round(d['ms_per_step'],3), 'ms/frame', {k:round(v,3) for k,v in d['kernel_ms_per_step'].items()}, 'eval kernel', round(d['roofline']['evals_per_s_kernel']/1e9,1))" || tail -3 gpurun_out/ab_$label.err
done
