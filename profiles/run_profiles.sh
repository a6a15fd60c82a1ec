# Round profile capture (run on a GPU box via gpurun from the repo root):
#   bash profiles/run_profiles.sh gpurun_out/vN
# tests, the bench line, the per-launch ncu list of one solve, ncu --set full
# of K6 (dominant), K5 and K6n, every config, the paper's experiments, multi-RHS
set -x
O=${1:-gpurun_out/prof}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; echo bench_rc=$?
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras"
timeout 300 $B > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lsqr_pipe -s 2 -c 1 -o $O/prof_k6 $B > $O/ncu_k6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_direct -c 1 -o $O/prof_k5 python profiles/time_api_sketch.py 40 > $O/ncu_k5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemv_rows -s 40 -c 1 -o $O/prof_k6n python profiles/time_alg1_arnoldi.py 60 > $O/ncu_k6n.log 2>&1
timeout 1500 python profiles/bench_configs.py c1 c2 c4 c3 c5 > $O/configs.jsonl 2> $O/configs.err
timeout 1500 python profiles/paper_experiments.py e5 e1 e4 > $O/paper_exp.jsonl 2> $O/paper_exp.err; echo pe_rc=$?
timeout 900 python profiles/bench_multirhs.py > $O/multirhs.jsonl 2> $O/multirhs.err
echo done
