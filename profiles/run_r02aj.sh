# CSR K1 block-boundary test; ncu of the c3 basis kernels (K1 stencil, K3) at the current build
O=gpurun_out/r02aj; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "boundaries or long_rows" --timeout 600 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR|E  )" $O/tests.log | head
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil_dots_v -s 50 -c 1 -o $O/prof_k1 $B > $O/ncu_k1.log 2>&1; echo k1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_tiles -s 50 -c 1 -o $O/prof_k3 $B > $O/ncu_k3.log 2>&1; echo k3_rc=$?
