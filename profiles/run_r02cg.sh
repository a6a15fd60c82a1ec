# multi-RHS CSR K1: resident CTAs per SM of the P > 1 instantiations (FAB_CSR_OCC_P 3 = default, 2, 4) at c4, p = 2 and 4
O=gpurun_out/r02cg; mkdir -p $O
timeout 1500 python profiles/csr_k1_ab.py c4 150 base1:default:1 base4:default:4 occp2_4:profiles/variants/libfab_occp2.so:4 occp4_4:profiles/variants/libfab_occp4.so:4 base2:default:2 occp2_2:profiles/variants/libfab_occp2.so:2 occp4_2:profiles/variants/libfab_occp4.so:2 > $O/csr_occp_ab_c4.jsonl 2> $O/ab.err; echo rc=$?
python -c "
import json
for l in open('$O/csr_occp_ab_c4.jsonl'):
    d=json.loads(l); print(d['variant'], d.get('p'), d.get('us_per_step_per_rhs'), d.get('H_sha'), d.get('error','')[:200])"
