cd $GRAFT_REPO_ROOT
O=gpurun_out/c65; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651"
timeout 300 $TR tools/mc_check.py > $O/mc_check.json 2> $O/mc_check.err
timeout 1200 python -m pytest tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest_exchange.log 2>&1; echo "rc=$?" >> $O/pytest_exchange.log
for P in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2966$P"
timeout 600 $TR bench.py --gpus $P --no-cpu-baseline --no-e2e > $O/bench_n$P.json 2> $O/bench_n$P.err
SG_PAYLOAD_MC=0 timeout 600 $TR bench.py --gpus $P --no-cpu-baseline --no-e2e > $O/bench_n${P}_nomc.json 2> $O/bench_n${P}_nomc.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671"
timeout 600 $TR bench.py --gpus 4 --no-cpu-baseline --no-e2e --cr 0.1 > $O/bench_n4_cr01.json 2> $O/bench_n4_cr01.err
timeout 600 $TR tools/multi_stress.py > $O/multi_stress.json 2> $O/multi_stress.err
