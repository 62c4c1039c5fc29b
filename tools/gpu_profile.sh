#!/bin/bash
# One GPU session: plain bench -> ncu launch list of one step -> ncu --set full of the first
# decoder layer's 7 launches.  Run under gpurun from the repo root.
set -x
OUT=gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json
$CMD > $OUT/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wl_gemv -s 1120 -c 224 --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain_small2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:wl_gemv -s 1120 -c 7 \
      -o $OUT/prof_stack $CMD > $OUT/ncu_full.log 2>&1
ls -la $OUT
