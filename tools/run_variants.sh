set -x
for v in base uncond rot n2 rotn2; do
  echo "== $v"
  WW_LIB_OVERRIDE=build/libww_$v.so python tools/chain_time.py 2048 2048 5504 2048 2048 5504 11008 2048
done
