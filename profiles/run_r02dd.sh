# K5 k_sketch_warp WITH the register prefetch at 12 warps per SM (accumulators in shared memory, sign words loaded late; 168 registers, 84-136 B of spills)
O=gpurun_out/r02dd; mkdir -p $O
for v in swa1o3 swa1w1o3; do
  FAB_LIB_VARIANT=profiles/variants/libfab_$v.so timeout 600 python profiles/k5_ab.py > $O/k5_ab_$v.jsonl 2> $O/$v.err; echo ${v}_rc=$?
done
timeout 600 python profiles/k5_ab.py > $O/k5_ab_base.jsonl 2> $O/base.err; echo base_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02dd/k5_ab_*.jsonl')):
    for l in open(f):
        d=json.loads(l)
        print(f.split('k5_ab_')[1][:-6], d['config'], {k:(round(d[k]['ms'],3), round(d[k]['gbs']), d[k]['maxrel_vs_fused']) for k in ('k_sketch_warp','k_sketch_direct','k_sketch_groups')})
PY
