# warp-block CSR K1 build variants (profiles/build_variant.py) vs the CTA kernel
O=gpurun_out/r02y; mkdir -p $O
V=profiles/variants
timeout 1800 python profiles/csr_k1_ab.py c4 150 base:default rp0:$V/libfab_rp0.so occ5:$V/libfab_occ5.so nb64:$V/libfab_nb64r32.so rp0occ5:$V/libfab_rp0occ5.so cta:default:1:FAB_CSR_K1=cta base2:default base_again:default > $O/ab_c4.jsonl 2> $O/ab_c4.err
timeout 1800 python profiles/csr_k1_ab.py c5 40 base:default rp0:$V/libfab_rp0.so occ5:$V/libfab_occ5.so nb64:$V/libfab_nb64r32.so cta:default:1:FAB_CSR_K1=cta > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for f in ['$O/ab_c4.jsonl','$O/ab_c5.jsonl']:
    for l in open(f):
        d=json.loads(l); print(d['config'], d['variant'], d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-200:])
"
