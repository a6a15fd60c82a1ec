# the bench's multi-GPU code path with one NCCL rank (torchrun, world 1) at the end-of-round build
O=gpurun_out/r02al; mkdir -p $O
FAB_BENCH_COMM=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_comm.json 2> $O/bench_comm.err; echo rc=$?
python -c "
import json;d=json.loads(open('$O/bench_comm.json').read().strip().splitlines()[-1]); print(d['value'], d['n_gpus'], d['config']['parallelism'], d.get('side_errors'), {c:d['configs'][c]['krylov_iters_per_s'] for c in d.get('configs',{})})"
