# warp-block CSR K1 final config: GPU suite, A/B vs CTA kernel, bench
O=gpurun_out/r02aa; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 1200 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR)" $O/tests.log | head
timeout 1800 python profiles/csr_k1_ab.py c4 150 warp:default cta:default:1:FAB_CSR_K1=cta warp2:default:2 cta2:default:2:FAB_CSR_K1=cta warp4:default:4 cta4:default:4:FAB_CSR_K1=cta > $O/ab_c4.jsonl 2> $O/ab_c4.err
timeout 1800 python profiles/csr_k1_ab.py c5 40 warp:default cta:default:1:FAB_CSR_K1=cta > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for f in ['$O/ab_c4.jsonl','$O/ab_c5.jsonl']:
    for l in open(f):
        d=json.loads(l); print(d['config'], d['variant'], d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-200:])
"
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
