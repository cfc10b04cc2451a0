#!/bin/bash
# Interleaved A/B of library builds / env knobs on the bench (no ncu), ROUNDS rounds.
# usage: tools/ab2.sh ROUNDS spec ...   spec = path/lib.so  or  label=path/lib.so:ENV=VAL[,ENV=VAL]
R=$1; shift
for r in $(seq 1 $R); do
  for spec in "$@"; do
    envs=""; lib=$spec; label=$(basename ${spec%%:*} .so)
    case $spec in *=*.so*) label=${spec%%=*}; lib=${spec#*=}; lib=${lib%%:*}; [[ $spec == *:* ]] && envs=${spec#*:};; esac
    label=${label}_$r
    env ${envs//,/ } PFT_LIB=$lib python bench.py --steps 20 --warmup ${AB_WARMUP:-3} --no-cpu-baseline --no-large > gpurun_out/ab_$label.json 2> gpurun_out/ab_$label.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_$label.json')); print('$label', round(d['value']/1e9,2), 'Gevals/s', round(d['ms_per_step'],4), 'ms/frame', {k:round(v,4) for k,v in d['kernel_ms_per_step'].items()}, 'eval', round(d['roofline']['evals_per_s_kernel']/1e9,1), 'agree', d.get('runs_agree'))" || tail -3 gpurun_out/ab_$label.err
  done
done
