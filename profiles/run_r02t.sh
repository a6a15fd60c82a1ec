O=gpurun_out/r02t; mkdir -p $O
./profiles/mtb_bin 300 > $O/micro_tma_box_sustained.jsonl; cut -c1-160 $O/micro_tma_box_sustained.jsonl | head -9
timeout 1500 python profiles/k6_rpl_ab.py c3 default: rpl2:FAB_LSQR_RPL=2,FAB_LSQR_KEEP=0 cl2:FAB_LSQR_CLUSTER=1 > $O/ab_c3.jsonl 2> $O/ab_c3.err
timeout 900 python profiles/k6_rpl_ab.py c2 default: rpl1:FAB_LSQR_RPL=1 rpl4:FAB_LSQR_RPL=4 > $O/ab_c2.jsonl 2> $O/ab_c2.err
timeout 900 python profiles/k6_rpl_ab.py c1 default: rpl1:FAB_LSQR_RPL=1 > $O/ab_c1.jsonl 2> $O/ab_c1.err
for f in $O/ab_*.jsonl; do python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(d['config'], d['variant'], round(d.get('ms_lsqr_pass',0),2), d.get('lsqr_iters'), round(d.get('ms_compress',0),2), d.get('error','')[-200:])"; done
