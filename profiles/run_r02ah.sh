O=gpurun_out/r02ah; mkdir -p $O
timeout 1800 python profiles/csr_k1_ab.py c5 40 p1:default:1 p1_persist:default:1:FAB_CSR_L2PERSIST=1 p1b:default:1 p1_persist_b:default:1:FAB_CSR_L2PERSIST=1 > $O/ab_c5.jsonl 2> $O/ab_c5.err
timeout 1800 python profiles/csr_k1_ab.py c4 150 p4:default:4 p4_persist:default:4:FAB_CSR_L2PERSIST=1 > $O/ab_c4.jsonl 2> $O/ab_c4.err
python -c "
import json
for f in ['$O/ab_c5.jsonl','$O/ab_c4.jsonl']:
  for l in open(f):
    d=json.loads(l); print(d['config'], d['variant'], d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('H_sha'), d.get('error','')[-300:])
"
