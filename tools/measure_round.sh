#!/bin/bash
# One GPU session that regenerates the round's committed measurements (run under gpurun from
# the repo root; everything lands in gpurun_out/round/, copied to profiles/<round>/): the
# default bench line, every config (C1-C3, C5 B=1..16), the decode-block chain and the
# persistent-program engine, the reference arm (the oracle), the O1-O4 / fusion ablations,
# the program's per-stage timeline, then the ncu launch list of one C4 step and a full ncu
# capture of one decoder layer (each ncu pass only after its command ran clean without ncu).
OUT=gpurun_out/round
mkdir -p $OUT
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python bench.py > $OUT/bench_c4_n1.json 2> $OUT/bench_c4_n1.err
: > $OUT/bench_engines.jsonl
for e in "--engine pdl --chain block" "--engine program --chain plain" "--engine program --chain block"; do
  python bench.py --steps 100 --no-cpu-baseline $e 2>> $OUT/bench_engines.err | tail -1 >> $OUT/bench_engines.jsonl
done
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
python tools/ablation_o1o4.py > $OUT/ablation_o1o4.txt 2>&1
python tools/prog_trace.py plain > $OUT/program_trace_plain.txt 2>&1
python tools/prog_trace.py block > $OUT/program_trace_block.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wl_gemv -s 512 -c 128 --csv \
      --log-file $OUT/ncu_launches_step.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain_small2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:wl_gemv -s 512 -c 4 \
      -o $OUT/prof_layer $CMD > $OUT/ncu_full.log 2>&1
ls -la $OUT
