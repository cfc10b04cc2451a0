#!/bin/bash
# writes profiles/r02_<tag>_* and the README / roofline-summary numbers from gpurun_out/*_<tag>* (after tools/round_check.sh <tag>)
T=$1; H=$(git rev-parse --short HEAD)
cp gpurun_out/bench_$T.json profiles/r02_${T}_bench.json; cp gpurun_out/ref_$T.json profiles/r02_${T}_reference.json
{ echo "# r02 $T build ($H): launch list of python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large"; echo "# ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 (cold-cache, serialised: compare shares; includes the map frames, the sweep, extraction and the F2/F2b emulations)"; python tools/ncu_summary.py launches gpurun_out/launches_$T.csv; } > profiles/r02_${T}_launches.txt
{ echo "# r02 $T ($H) k_track_persistent<float>: whole 10-iteration RO loop of a chained config-Q bench frame, one cooperative launch"; echo "# ncu --set full --clock-control none --import-source on -k regex:k_track_persistent -s 12 -c 1, python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-large; evals/launch = 2048 x 19200 x 10"; python tools/ncu_summary.py report gpurun_out/track_$T.ncu-rep 393216000; } > profiles/r02_${T}_track_ncu.txt
{ echo "# r02 $T ($H) k_integrate_list<float>, the 13th launch of the bench run (a warm-up frame of the chained config-Q sequence; ncu --set full --clock-control none, -s 12 -c 1)"; python tools/ncu_summary.py report gpurun_out/integ_$T.ncu-rep 1; } > profiles/r02_${T}_integrate_ncu.txt
python - "$T" <<'PY'
import json, re, sys
T = sys.argv[1]
tr = open(f'profiles/r02_{T}_track_ncu.txt').read()
rd = float(re.search(r'dram__bytes_read.sum\s+([\d.]+)', tr).group(1)); wr = float(re.search(r'dram__bytes_write.sum\s+([\d.]+)', tr).group(1))
b = (rd + wr) * 1e6 / 393216000
json.dump({"kernel": "k_track_persistent<float>", "dram_bytes_per_eval": b, "source": f"profiles/r02_{T}_track_ncu.txt: (dram__bytes_read.sum + dram__bytes_write.sum) of one k_track_persistent<float> launch (ncu --set full) / 2048 x 19200 x 10 evaluations"}, open('profiles/r02_track_traffic.json', 'w'), indent=1)
d = json.load(open(f'profiles/r02_{T}_bench.json'))
k = d['kernel_ms_per_step']; i = d['integration']; r = d['roofline']; L = d['large_volume']
hdr = ("# r02 final (%s) roofline summary — every kernel of the path, from profiles/r02_%s_*\n\n"
       "Numbers from `profiles/r02_%s_bench.json` (driver command `python bench.py --steps 20 --warmup 5`,\n"
       "CUDA-event times, L2 flushed between steps) and the ncu captures `profiles/r02_%s_*_ncu.txt` (extraction: `profiles/r02_v9_extract_ncu.txt`, kernel unchanged since).\n") % (T, T, T, T)
p = 'profiles/r02_roofline_summary.md'
s = open(p).read()
s = hdr + s[s.index("Peaks:"):]
s = re.sub(r"\| `k_track_persistent` \(a1-a9\), config Q \|.*\n", "| `k_track_persistent` (a1-a9), config Q | %.3f ms | 3.93e+08 evals x 32 B | gather (L2/L1) | %.0f GB/s | **%.2f** of the random-gather ceiling; %.3f of its own address stream's replay (3.61e+11 evals/s); DRAM %.0f MB/launch = %.3f B/eval (ncu, `profiles/r02_%s_track_ncu.txt`) |\n" % (k['track'], r['achieved'], r['frac'], r['gather_view']['frac'], rd + wr, b, T), s)
s = re.sub(r"\| `k_integrate_list` \(a10 fusion\), Q \| [\d.]+ us \| 1.98 M updated voxels x 16 B \| HBM \| \d+ GB/s \|", "| `k_integrate_list` (a10 fusion), Q | %.1f us | 1.98 M updated voxels x 16 B | HBM | %.0f GB/s |" % (i['us_fusion'], 16 * i['updated_voxels_per_frame'] / i['us_fusion'] / 1e3), s)
s = re.sub(r"\| cull \(frame prep \+ 2 levels\), Q \| [\d.]+ us \|", "| cull (frame prep + 2 levels), Q | %.1f us |" % i['us_cull'], s)
s = re.sub(r"\| `k_records_dirty` \(tracker records\), Q \| [\d.]+ us \|", "| `k_records_dirty` (tracker records), Q | %.1f us |" % i['us_records'], s)
s = re.sub(r"\| `k_track_persistent`, config L \(1024\^3 fp16, K = 4096\) \| [\d.]+ ms \| 7.86e\+08 evals \| gather \| — \| [\d.]+e\+11 evals/s \|", "| `k_track_persistent`, config L (1024^3 fp16, K = 4096) | %.3f ms | 7.86e+08 evals | gather | — | %.2fe+11 evals/s |" % (L['kernel_ms_per_frame']['track'], 7.86432e8 / L['kernel_ms_per_frame']['track'] / 1e8), s)
s = re.sub(r"Whole step: .*?; the tracker", "Whole step: %.3f ms per config-Q frame, %.3fe+11 evals/s (e2e with host I/O %.2fe+11); the tracker" % (d['ms_per_step'], d['value'] / 1e11, d['e2e']['value'] / 1e11), s)
open(p, 'w').write(s)
p = 'README.md'
s = open(p).read()
s = re.sub(r"round-2 final build, profiles/r02_v\d+_bench.json\)", "round-2 final build, profiles/r02_%s_bench.json)" % T, s)
s = re.sub(r"\*\*[\d.]+ ms/frame \(median [\d.]+\), [\d.]+e11 evals/s\*\* \(target: <5 ms, ≥1e11\); e2e with host I/O [\d.]+e11", "**%.3f ms/frame (median %.2f), %.3fe11 evals/s** (target: <5 ms, ≥1e11); e2e with host I/O %.2fe11" % (d['ms_per_step'], d['frame_ms']['median'], d['value'] / 1e11, d['e2e']['value'] / 1e11), s)
s = re.sub(r"\| [\d.]+ ms, [\d.]+e11 evals/s \|", "| %.3f ms, %.2fe11 evals/s |" % (k['track'], r['evals_per_s_kernel'] / 1e11), s)
s = re.sub(r"at the band's footprint \(8.79 TB/s\): \*\*[\d.]+\*\*", "at the band's footprint (8.79 TB/s): **%.2f**" % r['frac'], s)
s = re.sub(r"on-device regeneration\): [\d.]+ for the whole", "on-device regeneration): %.3f for the whole" % r['gather_view']['frac'], s)
open(p, 'w').write(s)
print(d['value'], d['ms_per_step'])
PY
