set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/c2; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py -m gpu -x -q -rs > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 600 $TR bench.py --gpus $N --no-e2e > $O/bench_n${N}.json 2> $O/bench_n${N}.err
timeout 600 $TR bench.py --gpus $N --no-e2e --cr 0.001 > $O/bench_n${N}_cr0001.json 2> $O/bench_n${N}_cr0001.err
timeout 600 $TR bench.py --gpus $N --no-e2e --workload dense > $O/bench_n${N}_dense.json 2> $O/bench_n${N}_dense.err
timeout 600 $TR bench.py --gpus $N --no-e2e --family mixed > $O/bench_n${N}_mixed.json 2> $O/bench_n${N}_mixed.err
timeout 600 $TR bench.py --gpus $N --no-e2e --cr 0.1 > $O/bench_n${N}_cr01.json 2> $O/bench_n${N}_cr01.err
ls -la $O
