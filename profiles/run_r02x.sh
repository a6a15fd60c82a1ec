# Warp-block CSR K1 v2 (headers one block ahead, row pointers issued with the entries)
O=gpurun_out/r02x; mkdir -p $O
timeout 1500 python profiles/csr_k1_ab.py c4 150 warp:default cta:default:1:FAB_CSR_K1=cta warp4:default:4 cta4:default:4:FAB_CSR_K1=cta warp2:default:2 cta2:default:2:FAB_CSR_K1=cta > $O/ab_c4.jsonl 2> $O/ab_c4.err; cut -c1-200 $O/ab_c4.jsonl
timeout 1500 python profiles/csr_k1_ab.py c5 40 warp:default cta:default:1:FAB_CSR_K1=cta > $O/ab_c5.jsonl 2> $O/ab_c5.err; cut -c1-200 $O/ab_c5.jsonl
timeout 1800 python -m pytest tests/test_gpu_parity_large_m.py tests/test_gpu_batch.py tests/test_gpu_csr_plan.py tests/test_gpu_golden_c4.py tests/test_gpu_fullsize_csr.py tests/test_gpu_loopback.py -m gpu -q --timeout 1200 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR)" $O/tests.log | head
