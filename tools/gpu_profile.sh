#!/bin/bash
# One GPU session: plain bench -> ncu launch list of one C4 step (128 launches: qkv, o,
# gate/up, down x 32 layers) -> ncu --set full of one decoder layer's 4 launches.
# Run under gpurun from the repo root; writes gpurun_out/.
set -x
OUT=gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json
# warm-up eager steps (3) + the eager step before capture = 4 x 128 launches to skip
$CMD > $OUT/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wl_gemv -s 512 -c 128 --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain_small2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:wl_gemv -s 512 -c 4 \
      -o $OUT/prof_stack $CMD > $OUT/ncu_full.log 2>&1
ls -la $OUT
