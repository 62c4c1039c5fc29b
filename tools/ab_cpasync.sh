for mode in 0 1; do
python - <<PY
import os, sys, json, subprocess
sys.argv=['bench.py','--steps','50','--warmup','5','--no-cpu-baseline']
import paper_2604_20913_b200 as ww
ww._lib.ww_debug_force_cp_async($mode)
import bench, io, contextlib
buf=io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d=json.loads(buf.getvalue().strip().splitlines()[-1])
print("force_cp_async=$mode", d["ms_per_step"], d["per_shape_us"])
PY
done
