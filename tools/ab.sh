#!/bin/bash
# A/B of library builds on the default bench (ms per token) and per-shape PDL chains.
# usage: tools/ab.sh name=lib.so [name=lib.so ...]   (lib "" = the in-tree product build)
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  WW_LIB_OVERRIDE=$lib python bench.py --steps 100 --no-cpu-baseline > gpurun_out/ab_$name.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name', d['ms_per_step'], d['per_shape_us'])"
done
