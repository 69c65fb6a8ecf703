cd $GRAFT_REPO_ROOT
O=gpurun_out/c19; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 300 $TR tools/dense_timing.py > $O/dense_nvls.json 2> $O/dense_nvls.err
timeout 900 python -m pytest tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 $TR bench.py --gpus $N --no-e2e --workload dense > $O/bench_n${N}_dense.json 2> $O/bench_n${N}_dense.err
