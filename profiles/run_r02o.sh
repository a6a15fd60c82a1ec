O=gpurun_out/r02o; mkdir -p $O
timeout 1500 python profiles/k6_rpl_ab.py c3 nocl:FAB_LSQR_CLUSTER=0 cl:FAB_LSQR_CLUSTER=1 cl_rpl1:FAB_LSQR_CLUSTER=1,FAB_LSQR_RPL=1 nocl_b:FAB_LSQR_CLUSTER=0 cl_b:FAB_LSQR_CLUSTER=1 > $O/ab_c3.jsonl 2> $O/ab_c3.err
cut -c1-250 $O/ab_c3.jsonl; tail -3 $O/ab_c3.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large_m.py tests/test_gpu_lsqr_graph.py tests/test_gpu_async.py -q --timeout 600 -p no:cacheprovider > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
tail -2 $O/tests.log; grep -E "^FAILED|^ERROR|^E  " $O/tests.log | head -20
