# A/B of library builds on the C5 batched variant (bench --workload c5), us per layer
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  for b in 4 8 16; do
    WW_LIB_OVERRIDE=$lib python bench.py --workload c5 --batch $b --steps 50 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$name', 'B=$b', d['us_per_layer'], d['alu_frac'])"
  done
done
