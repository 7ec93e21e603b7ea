#!/usr/bin/env bash
# Round-end measurement set (run on the GPU box via gpurun; outputs in gpurun_out/prof/):
# bench lines for every BASELINE config that fits one GPU, both propagators, the
# reference arm, an ncu launch list and ncu --set full captures of the step
# kernels at 240^3, 512^3 (r = 2, 4, 8) and 1000^3 (each command first ran
# plain and exited 0: bench lines before the captures).
set -u
O=gpurun_out/prof
mkdir -p $O
b() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; }
if [ "${1:-}" != "--ncu-only" ]; then
b bench_240
b bench_512 --grid 512 --steps 200
b bench_1000 --grid 1000 --steps 40 --warmup 5
b bench_512_r2 --grid 512 --radius 2 --steps 200
b bench_512_r8 --grid 512 --radius 8 --steps 100
b bench_vd_240 --propagator acoustic_iso
b bench_reference_240 --impl reference --steps 20 --warmup 3
b bench_reference_1000 --impl reference --scaling strong --steps 2 --warmup 1
fi
[ "${1:-}" = "--no-ncu" ] && exit 0
P="python tools/cpml_probe.py --steps 5"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_240.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
for g in 240 512 1000; do
  $P --grid $g > $O/plain_$g.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_bnd|k_p1|k_inner|k_zslab' \
      -s 24 -c 4 -o $O/full_$g -f $P --grid $g > $O/ncu_full_$g.log 2>&1
  echo "ncu full $g rc=$?"
done
for r in 2 8; do
  $P --grid 512 --radius $r > $O/plain_512_r$r.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_bnd|k_p1|k_inner|k_zslab' \
      -s 24 -c 4 -o $O/full_512_r$r -f $P --grid 512 --radius $r > $O/ncu_full_512_r$r.log 2>&1
  echo "ncu full 512 r$r rc=$?"
done
$P --grid 240 --variants "cpml_fused=1" > $O/plain_cpml.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_cpml' -s 12 -c 1 \
    -o $O/full_cpml_240 -f $P --grid 240 --variants "cpml_fused=1" > $O/ncu_cpml.log 2>&1
echo "ncu cpml rc=$?"
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
# gpurun brings back at most 64 MiB: keep the raw exports, drop the large reports
find $O -name '*.ncu-rep' -size +12M -delete
du -sh $O
echo done
