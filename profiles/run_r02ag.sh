O=gpurun_out/r02ag; mkdir -p $O
timeout 1800 python profiles/csr_k1_ab.py c4 150 p4:default:4 p4_f40:default:4:FAB_BATCH_BLOCKFRAC=0.4 p3:default:3 p2:default:2 > $O/ab_c4.jsonl 2> $O/ab_c4.err
timeout 1800 python profiles/csr_k1_ab.py c5 20 p1:default:1 p2:default:2 p2_f40:default:2:FAB_BATCH_BLOCKFRAC=0.4 p4:default:4 p4_f40:default:4:FAB_BATCH_BLOCKFRAC=0.4 > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for f in ['$O/ab_c4.jsonl','$O/ab_c5.jsonl']:
  for l in open(f):
    d=json.loads(l); print(d['config'], d['variant'], d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-300:])
"
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q --timeout 600 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -2 $O/tests.log
