# Round profile capture (run on a GPU box via gpurun from the repo root):
#   tests, full bench line, per-launch ncu list of one solve, ncu --set full of the three streaming kernels
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo tests_rc=$? >> gpurun_out/tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
for K in k_lsqr_pipe k_stream_tiles k_stencil_dots_v; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$K $B > gpurun_out/ncu_$K.log 2>&1
done
echo done
