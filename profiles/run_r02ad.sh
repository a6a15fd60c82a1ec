# c5: old z prefetched before the gathers in the z += passes (new) vs committed (old); c5 golden test
O=gpurun_out/r02ad; mkdir -p $O
V=profiles/variants
timeout 1800 python profiles/csr_k1_ab.py c5 40 new:default old:$V/libfab_old.so new2:default old2:$V/libfab_old.so > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for l in open('$O/ab_c5.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], round(d.get('us_per_step_per_rhs',0),1), d.get('H_sha'), d.get('error','')[-300:])
"
timeout 1800 python -m pytest tests/test_gpu_golden_c5.py tests/test_gpu_golden_c4.py -m gpu -q --timeout 1500 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR|E )" $O/tests.log | head -20
