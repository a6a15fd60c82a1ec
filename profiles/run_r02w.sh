# Warp-block CSR K1 (k_csr_warp, default) vs the CTA-block k_csr_stream
# (FAB_CSR_K1=cta): GPU suite, c4 / c5 A/B per Krylov step, ncu of c4's K1.
O=gpurun_out/r02w; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 1200 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR)" $O/tests.log | head
timeout 1500 python profiles/csr_k1_ab.py c4 150 warp:default cta:default:1:FAB_CSR_K1=cta warp4:default:4 cta4:default:4:FAB_CSR_K1=cta warp2:default:2 > $O/ab_c4.jsonl 2> $O/ab_c4.err; cut -c1-200 $O/ab_c4.jsonl
timeout 1500 python profiles/csr_k1_ab.py c5 40 warp:default cta:default:1:FAB_CSR_K1=cta > $O/ab_c5.jsonl 2> $O/ab_c5.err; cut -c1-200 $O/ab_c5.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_warp -s 3 -c 1 -o $O/prof_c4_warp python profiles/csr_k1_driver.py c4 1 > $O/ncu_c4.log 2>&1; echo ncu_rc=$?
