# K5 k_sketch_warp timing-only diagnostics (values wrong by construction): where the 7.6 ms go -- butterflies, exchange, or the load path
O=gpurun_out/r02dc; mkdir -p $O
for v in swt1 swt2 swt2o4; do
  FAB_LIB_VARIANT=profiles/variants/libfab_$v.so timeout 600 python profiles/k5_ab.py > $O/k5_ab_$v.jsonl 2> $O/$v.err; echo ${v}_rc=$?
done
timeout 600 python profiles/k5_ab.py > $O/k5_ab_base.jsonl 2> $O/base.err; echo base_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02dc/k5_ab_*.jsonl')):
    for l in open(f):
        d=json.loads(l)
        print(f.split('k5_ab_')[1][:-6], d['config'], {k:(round(d[k]['ms'],3), round(d[k]['gbs'])) for k in ('k_sketch_warp','k_sketch_direct','k_sketch_groups')})
PY
