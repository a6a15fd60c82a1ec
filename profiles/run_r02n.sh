O=gpurun_out/r02n; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large_m.py tests/test_gpu_lsqr_graph.py tests/test_gpu_async.py -q --timeout 600 -p no:cacheprovider > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
tail -2 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head
timeout 1500 python profiles/k6_rpl_ab.py c3 rpl1:FAB_LSQR_RPL=1 rpl2keep:FAB_LSQR_RPL=2,FAB_LSQR_KEEP=1 rpl2nokeep:FAB_LSQR_RPL=2,FAB_LSQR_KEEP=0 default: > $O/ab_c3.jsonl 2> $O/ab_c3.err
cut -c1-330 $O/ab_c3.jsonl
timeout 900 python profiles/k6_rpl_ab.py c2 rpl1:FAB_LSQR_RPL=1 rpl2:FAB_LSQR_RPL=2 rpl4keep:FAB_LSQR_RPL=4,FAB_LSQR_KEEP=1 rpl4nokeep:FAB_LSQR_RPL=4,FAB_LSQR_KEEP=0 > $O/ab_c2.jsonl 2> $O/ab_c2.err
cut -c1-330 $O/ab_c2.jsonl
