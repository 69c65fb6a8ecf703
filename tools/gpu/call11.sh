cd $GRAFT_REPO_ROOT
O=gpurun_out/c11; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/topk_timing.py --crs 0.01,0.1 > $O/topk_chain.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 300 $TR tools/dense_timing.py > $O/dense_push.json 2> $O/dense_push.err
SG_DENSE_PULL=1 timeout 300 $TR tools/dense_timing.py > $O/dense_pull.json 2> $O/dense_pull.err
timeout 600 $TR bench.py --gpus $N --no-e2e > $O/bench_n$N.json 2> $O/bench_n$N.err
timeout 600 $TR bench.py --gpus $N --no-e2e --cr 0.001 > $O/bench_n${N}_cr0001.json 2> $O/bench_n${N}_cr0001.err
timeout 600 $TR bench.py --gpus $N --no-e2e --workload dense > $O/bench_n${N}_dense.json 2> $O/bench_n${N}_dense.err
timeout 600 $TR bench.py --gpus $N --no-e2e --family mixed > $O/bench_n${N}_mixed.json 2> $O/bench_n${N}_mixed.err
