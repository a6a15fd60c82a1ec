O=gpurun_out/r02af; mkdir -p $O
timeout 1800 python profiles/csr_k1_ab.py c4 150 p4_3blk:default:4 p4_unblocked:default:4:FAB_BATCH_L2FRAC=1.2 p4_2blk:default:4:FAB_BATCH_COLBLOCK=2097152 p4_4blk:default:4:FAB_BATCH_COLBLOCK=1048576 p2:default:2 p3:default:3 p1:default:1 > $O/ab_c4.jsonl 2> $O/ab_c4.err
python -c "
import json
for l in open('$O/ab_c4.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], d.get('p'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-300:])
"
