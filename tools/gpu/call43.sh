cd $GRAFT_REPO_ROOT
O=gpurun_out/c43; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > $O/topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py -m gpu -x -q -rs > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
for P in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2960$P"
timeout 600 $TR bench.py --gpus $P > $O/bench_n$P.json 2> $O/bench_n$P.err
timeout 600 $TR bench.py --gpus $P --impl reference > $O/bench_ref_n$P.json 2> $O/bench_ref_n$P.err
timeout 600 $TR bench.py --gpus $P --no-e2e --cr 0.001 > $O/bench_n${P}_cr0001.json 2> $O/bench_n${P}_cr0001.err
timeout 600 $TR bench.py --gpus $P --no-e2e --cr 0.1 > $O/bench_n${P}_cr01.json 2> $O/bench_n${P}_cr01.err
timeout 600 $TR bench.py --gpus $P --no-e2e --workload dense > $O/bench_n${P}_dense.json 2> $O/bench_n${P}_dense.err
timeout 600 $TR bench.py --gpus $P --no-e2e --family mixed > $O/bench_n${P}_mixed.json 2> $O/bench_n${P}_mixed.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29610"
for mode in pull push nvls fused; do SG_DENSE_MODE=$mode timeout 300 $TR tools/dense_timing.py > $O/dense_$mode.json 2> $O/dense_$mode.err; done
timeout 600 $TR tools/shard_tradeoff.py > $O/shard.json 2> $O/shard.err
timeout 600 $TR tools/multi_check.py > $O/multi_check.json 2> $O/multi_check.err
SG_CHECK_WORKERS=4 timeout 600 $TR tools/multi_check.py > $O/multi_check_w4.json 2> $O/multi_check_w4.err
timeout 900 $TR tools/train_resnet152.py --steps 4 > $O/train_n4.json 2> $O/train_n4.err
