O=gpurun_out/r02r; mkdir -p $O
timeout 1500 python profiles/k6_rpl_ab.py c3 cl2:FAB_LSQR_CLUSTER=1 cl1:FAB_LSQR_CLUSTER=1,FAB_LSQR_RPL=1 rpl1:FAB_LSQR_CLUSTER=0,FAB_LSQR_RPL=1 > $O/ab_c3.jsonl 2> $O/ab_c3.err
cut -c1-250 $O/ab_c3.jsonl; tail -3 $O/ab_c3.err
FAB_LSQR_CLUSTER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lsqr_pipe_cl -s 3 -c 1 -o $O/k6cl2 python profiles/k6_rpl_ab.py --child c3 > $O/ncu.log 2>&1; echo ncu_rc=$?; tail -1 $O/ncu.log
timeout 600 python -m pytest tests/test_gpu_parity_large_m.py tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -x > $O/tests.log 2>&1; echo rc=$?; tail -3 $O/tests.log
