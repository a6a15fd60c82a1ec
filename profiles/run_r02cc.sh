# K5 as warp sub-tiles (k_sketch_warp): parity tests, A/B timing, ncu of the c3 pass
O=gpurun_out/r02cc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch or k5" --timeout 600 > $O/tests_k5.log 2>&1; echo tests_k5_rc=$?; tail -3 $O/tests_k5.log
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_dist.py tests/test_gpu_batch.py tests/test_gpu_parity_large_m.py -q -x --timeout 600 > $O/tests_users.log 2>&1; echo tests_users_rc=$?; tail -3 $O/tests_users.log
timeout 900 python profiles/k5_ab.py > $O/k5_ab.jsonl 2> $O/k5_ab.err; echo ab_rc=$?; cat $O/k5_ab.jsonl
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sketch_bulk -c 1 -o $O/k5_bulk_c3 python profiles/k5_ncu_driver.py > $O/ncu.log 2>&1; echo ncu_rc=$?
ncu -i $O/k5_bulk_c3.ncu-rep --page details --csv > $O/k5_bulk_c3_details.csv 2>/dev/null; grep -E "Duration|DRAM Throughput|Memory Throughput|L1/TEX Hit|Registers|Achieved Occupancy" $O/k5_bulk_c3_details.csv | head -12
