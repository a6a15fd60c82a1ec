# c5 column-block width sweep with the warp-block K1; ncu of k_csr_warp (c4, c5)
O=gpurun_out/r02ac; mkdir -p $O
timeout 1800 python profiles/csr_k1_ab.py c5 40 w6:default w4:default:1:FAB_CSR_COLBLOCK=8388608 w8:default:1:FAB_CSR_COLBLOCK=4194304 w3:default:1:FAB_CSR_COLBLOCK=11184811 w12:default:1:FAB_CSR_COLBLOCK=2796203 > $O/ab_c5.jsonl 2> $O/ab_c5.err
python -c "
import json
for l in open('$O/ab_c5.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], d.get('env'), round(d.get('us_per_step_per_rhs',0),1), d.get('error','')[-300:])
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_warp -s 3 -c 1 -o $O/prof_c4_warp python profiles/csr_k1_driver.py c4 1 > $O/ncu_c4.log 2>&1; echo ncu4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_warp -s 7 -c 2 -o $O/prof_c5_warp python profiles/csr_k1_driver.py c5 1 > $O/ncu_c5.log 2>&1; echo ncu5_rc=$?
