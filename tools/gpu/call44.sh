cd $GRAFT_REPO_ROOT
O=gpurun_out/c44; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR tools/multi_check.py > $O/multi_check.json 2> $O/multi_check.err
for c in 1 2 4 8 16; do SG_DENSE_CHUNKS=$c timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --workload dense > $O/dense_c$c.json 2> $O/dense_c$c.err; done
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612"
for c in 1 4 8; do SG_DENSE_CHUNKS=$c CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --no-e2e --no-cpu-baseline --workload dense > $O/dense2_c$c.json 2> $O/dense2_c$c.err; done
