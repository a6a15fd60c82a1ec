O=gpurun_out/r02l; mkdir -p $O
V=profiles/variants
timeout 2400 python profiles/csr_k1_ab.py c4 150 p1:default:1 p4blk:default:4 p4one:default:4:FAB_BATCH_L2FRAC=1.2 p4blk_occ4:$V/libfab_occp4.so:4 p4one_occ4:$V/libfab_occp4.so:4:FAB_BATCH_L2FRAC=1.2 p4blk_occ2:$V/libfab_occp2.so:4 p2blk:default:2:FAB_BATCH_L2FRAC=0.3 p2one:default:2 p2one_occ4:$V/libfab_occp4.so:2 > $O/ab_c4.jsonl 2> $O/ab_c4.err
cut -c1-120 $O/ab_c4.jsonl; python -c "
import json
for l in open('$O/ab_c4.jsonl'):
    d=json.loads(l); print(d.get('variant'), d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-200:])"
