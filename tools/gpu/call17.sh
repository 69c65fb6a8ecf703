cd $GRAFT_REPO_ROOT
O=gpurun_out/c17; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 300 $TR tools/dense_timing.py > $O/dense_nvls.json 2> $O/dense_nvls.err
timeout 900 python -m pytest tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 $TR bench.py --gpus $N --no-e2e --workload dense > $O/bench_n${N}_dense.json 2> $O/bench_n${N}_dense.err
timeout 600 $TR bench.py --gpus $N --no-e2e --cr 0.001 > $O/bench_n${N}_cr0001.json 2> $O/bench_n${N}_cr0001.err
timeout 600 $TR bench.py --gpus $N --no-e2e --family mixed > $O/bench_n${N}_mixed.json 2> $O/bench_n${N}_mixed.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/topk_timing.py --ks 1,2,8 > $O/topk_chain.txt 2>&1
