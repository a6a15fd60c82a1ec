O=gpurun_out/r02ae; mkdir -p $O
V=profiles/variants
timeout 1800 python profiles/csr_k1_ab.py c4 150 base:default nb256:$V/libfab_nb256.so nb256r128:$V/libfab_nb256r128.so > $O/ab_c4.jsonl 2> $O/ab_c4.err
timeout 1800 python profiles/csr_k1_ab.py c5 40 base:default nb256:$V/libfab_nb256.so nb256r128:$V/libfab_nb256r128.so > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for f in ['$O/ab_c4.jsonl','$O/ab_c5.jsonl']:
  for l in open(f):
    d=json.loads(l); print(d['config'], d['variant'], round(d.get('us_per_step_per_rhs',0),1), d.get('H_sha'), d.get('error','')[-300:])
"
