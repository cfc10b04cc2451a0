#!/bin/bash
# round-end verification on one B200: GPU tests, smoke, bench + reference arm, launch list, ncu captures
T=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/tests_$T.txt; cat gpurun_out/tests_$T.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large > gpurun_out/ncu_l_$T.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --clock-control none --import-source on -k "regex:k_track_persistent" -s 12 -c 1 -o gpurun_out/track_$T python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large > gpurun_out/ncu_t_$T.log 2>&1; echo ncu_track_rc=$?
ncu --set full --clock-control none --import-source on -k "regex:k_integrate_list" -s 12 -c 1 -o gpurun_out/integ_$T python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large > gpurun_out/ncu_i_$T.log 2>&1; echo ncu_integ_rc=$?
