O=gpurun_out/r02k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_csr_plan.py tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -x > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
tail -2 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head
V=profiles/variants
timeout 1200 python profiles/csr_k1_ab.py c4 150 pre6:default base:$V/libfab_base.so pre5:$V/libfab_pre5.so nopre5:$V/libfab_nopre5.so pre4:$V/libfab_pre4.so pre6b:default base_b:$V/libfab_base.so > $O/ab_c4.jsonl 2> $O/ab_c4.err
cat $O/ab_c4.jsonl | cut -c1-200
timeout 1500 python profiles/csr_k1_ab.py c5 40 pre6:default base:$V/libfab_base.so pre5:$V/libfab_pre5.so > $O/ab_c5.jsonl 2> $O/ab_c5.err
cat $O/ab_c5.jsonl | cut -c1-200
