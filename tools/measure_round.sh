#!/bin/bash
# One GPU session that regenerates the round's committed measurements (run under gpurun from
# the repo root; everything lands in gpurun_out/round/, copied to profiles/<round>/ by hand):
# default bench line, every config (C1-C3, C5 B=1..16), the reference arm (the oracle), the
# seed CV of per-layer times, the unfused ablation, then the ncu launch list of one C4 step
# and a full ncu capture of one decoder layer (each ncu pass only after its command ran
# clean without ncu).
OUT=gpurun_out/round
mkdir -p $OUT
set -x
python bench.py > $OUT/bench_c4_n1.json 2> $OUT/bench_c4_n1.err
: > $OUT/bench_configs.jsonl
for w in c1 c2 c3a c3b; do
  python bench.py --workload $w --steps 50 --no-cpu-baseline 2>> $OUT/bench_configs.err \
    | tail -1 >> $OUT/bench_configs.jsonl
done
for b in 1 2 4 8 16; do
  python bench.py --workload c5 --batch $b --steps 50 --no-cpu-baseline 2>> $OUT/bench_configs.err \
    | tail -1 >> $OUT/bench_configs.jsonl
done
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_arm.json 2>&1
python tools/seed_cv.py > $OUT/seed_cv.txt 2>&1
python tools/ablation_unfused.py > $OUT/ablation_unfused.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wl_gemv -s 512 -c 128 --csv \
      --log-file $OUT/ncu_launches_step.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain_small2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:wl_gemv -s 512 -c 4 \
      -o $OUT/prof_layer $CMD > $OUT/ncu_full.log 2>&1
ls -la $OUT
