# K5 v3 k_sketch_warp build-time variants (no register prefetch / accumulators in shared memory / 3-4 CTAs per SM) against the in-tree kernels, c2 and c3
O=gpurun_out/r02db; mkdir -p $O
timeout 600 python profiles/k5_ab.py > $O/k5_ab_base.jsonl 2> $O/base.err; echo base_rc=$?
for v in swpf0o3 swpf0a1o3 swpf0a1o4; do
  FAB_LIB_VARIANT=profiles/variants/libfab_$v.so timeout 600 python profiles/k5_ab.py > $O/k5_ab_$v.jsonl 2> $O/$v.err; echo ${v}_rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02db/k5_ab_*.jsonl')):
    for l in open(f):
        d=json.loads(l)
        print(f.split('k5_ab_')[1][:-6], d['config'], {k:(round(d[k]['ms'],3), round(d[k]['gbs']), d[k]['maxrel_vs_fused']) for k in ('k_sketch_warp','k_sketch_direct','k_sketch_groups')})
PY
FAB_SKETCH_K5=3 FAB_LIB_VARIANT=profiles/variants/libfab_swpf0a1o4.so timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or k5 or K5" > $O/tests_k5_swpf0a1o4.log 2>&1; tail -2 $O/tests_k5_swpf0a1o4.log
