cd $GRAFT_REPO_ROOT
O=gpurun_out/c16; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 300 $TR tools/dense_timing.py > $O/dense_fused.json 2> $O/dense_fused.err
SG_DENSE_MODE=push timeout 300 $TR tools/dense_timing.py > $O/dense_push.json 2> $O/dense_push.err
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py tests/test_gpu_topk.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 $TR bench.py --gpus $N --no-e2e --workload dense > $O/bench_n${N}_dense.json 2> $O/bench_n${N}_dense.err
timeout 600 $TR bench.py --gpus $N --no-e2e --cr 0.001 > $O/bench_n${N}_cr0001.json 2> $O/bench_n${N}_cr0001.err
timeout 600 $TR bench.py --gpus $N --no-e2e --family mixed > $O/bench_n${N}_mixed.json 2> $O/bench_n${N}_mixed.err
timeout 600 $TR bench.py --gpus $N --no-e2e > $O/bench_n$N.json 2> $O/bench_n$N.err
timeout 300 $TR tools/shard_tradeoff.py > $O/shard.json 2> $O/shard.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/topk_timing.py --ks 1,8 > $O/topk_chain.txt 2>&1
