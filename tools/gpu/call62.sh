cd $GRAFT_REPO_ROOT
O=gpurun_out/c62; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py -m gpu -x -q -rs > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
for P in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2960$P"
timeout 600 $TR bench.py --gpus $P --no-cpu-baseline > $O/bench_n$P.json 2> $O/bench_n$P.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --cr 0.001 > $O/bench_n4_cr0001.json 2> $O/bench_n4_cr0001.err
timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --cr 0.1 > $O/bench_n4_cr01.json 2> $O/bench_n4_cr01.err
timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --workload dense > $O/bench_n4_dense.json 2> $O/bench_n4_dense.err
timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --family mixed > $O/bench_n4_mixed.json 2> $O/bench_n4_mixed.err
timeout 600 $TR tools/shard_tradeoff.py > $O/shard.json 2> $O/shard.err
timeout 600 $TR tools/multi_check.py > $O/multi_check.json 2> $O/multi_check.err
timeout 600 $TR tools/multi_stress.py > $O/multi_stress.json 2> $O/multi_stress.err
timeout 600 $TR tools/config4.py > $O/config4_n4.json 2> $O/config4_n4.err
