# Round-2 capture (run on a GPU box via gpurun from the repo root):
#   bash profiles/run_r02.sh gpurun_out/r02a [tests|notests]
# GPU tests, the driver's bench command, the per-launch ncu list of one bench
# step (gpu__time_duration / dram bytes per launch), ncu --set full of K6 (the
# dominant kernel: traffic for roofline.traffic) and of both K5 kernels.
set -x
O=${1:-gpurun_out/r02}
mkdir -p $O
if [ "${2:-tests}" = "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
fi
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --no-configs"
timeout 300 $B > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lsqr_pipe -s 2 -c 1 -o $O/prof_k6 $B > $O/ncu_k6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_direct -c 1 -o $O/prof_k5 python profiles/time_api_sketch.py 40 > $O/ncu_k5.log 2>&1
FAB_SKETCH_K5=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_groups -c 1 -o $O/prof_k5g python profiles/time_api_sketch.py 40 > $O/ncu_k5g.log 2>&1
echo done
