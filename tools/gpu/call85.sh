cd $GRAFT_REPO_ROOT
O=gpurun_out/c85; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py -m gpu -x -q -rs > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
for P in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2985$P"
timeout 600 $TR bench.py --gpus $P > $O/bench_n$P.json 2> $O/bench_n$P.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29861"
for cr in 0.1 0.001; do timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --cr $cr > $O/bench_n4_cr$cr.json 2> $O/bench_n4_cr$cr.err; done
timeout 600 $TR bench.py --gpus 4 --no-e2e --no-cpu-baseline --workload dense > $O/bench_n4_dense.json 2> $O/bench_n4_dense.err
timeout 600 $TR bench.py --gpus 4 --workers 4 --no-cpu-baseline --no-e2e > $O/bench_n4_w4.json 2> $O/bench_n4_w4.err
timeout 600 $TR tools/multi_stress.py --steps 60 > $O/multi_stress.json 2> $O/multi_stress.err
timeout 600 $TR tools/config4.py > $O/config4_n4.json 2> $O/config4_n4.err
