O=gpurun_out/r02s; mkdir -p $O
FAB_VERBOSE=1 timeout 1500 python profiles/k6_rpl_ab.py c3 cl2:FAB_LSQR_CLUSTER=1,FAB_VERBOSE=1 rpl1:FAB_LSQR_CLUSTER=0,FAB_LSQR_RPL=1 > $O/ab_c3.jsonl 2> $O/ab_c3.err
cut -c1-250 $O/ab_c3.jsonl; grep -h 'fab\]' $O/ab_c3.err | head -3
