#!/usr/bin/env bash
# Round-end measurement set (run on the GPU box via gpurun; outputs in gpurun_out/prof/):
# bench lines for every BASELINE config that fits one GPU, both propagators, the
# reference arm, an ncu launch list and one ncu --set full capture of the step kernels.
set -u
O=gpurun_out/prof
mkdir -p $O
b() { local name=$1; shift; python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; }
b bench_240
b bench_512 --grid 512 --steps 200
b bench_1000 --grid 1000 --steps 40 --warmup 5
b bench_512_r2 --grid 512 --radius 2 --steps 200
b bench_512_r8 --grid 512 --radius 8 --steps 100
b bench_vd_240 --propagator acoustic_iso
b bench_vd_512 --propagator acoustic_iso --grid 512 --steps 100
b bench_vd_1000 --propagator acoustic_iso --grid 1000 --steps 20 --warmup 3
b bench_reference_240 --impl reference --steps 20 --warmup 3
b bench_vd_reference_240 --impl reference --propagator acoustic_iso --steps 20 --warmup 3
[ "${1:-}" = "--no-ncu" ] && exit 0
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_240.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k 'regex:k_bnd|k_p1|k_inner' -s 60 -c 4 \
    -o $O/full_240 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i $O/full_240.ncu-rep --page raw --csv > $O/full_240_raw.csv 2>/dev/null
