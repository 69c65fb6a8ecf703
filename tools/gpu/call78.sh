cd $GRAFT_REPO_ROOT
O=gpurun_out/c78; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801"
timeout 300 $TR tools/multi_stress.py --steps 60 > $O/multi_stress.json 2> $O/multi_stress.err
timeout 300 $TR tools/multi_timing.py > $O/timing_n4.json 2> $O/timing_n4.err
for pb in 1 0; do SG_PEER_BARRIER=$pb timeout 300 $TR bench.py --gpus 4 --no-cpu-baseline --no-e2e > $O/bench_n4_pb$pb.json 2> $O/bench_n4_pb$pb.err; done
for pb in 1 0; do SG_PEER_BARRIER=$pb timeout 300 $TR bench.py --gpus 4 --no-cpu-baseline --no-e2e --family mixed > $O/bench_n4_mixed_pb$pb.json 2> $O/bench_n4_mixed_pb$pb.err; done
timeout 300 $TR bench.py --gpus 4 --workers 4 --no-cpu-baseline --no-e2e > $O/bench_n4_w4.json 2> $O/bench_n4_w4.err
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29802"
for pb in 1 0; do SG_PEER_BARRIER=$pb CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR2 bench.py --gpus 2 --no-cpu-baseline --no-e2e > $O/bench_n2_pb$pb.json 2> $O/bench_n2_pb$pb.err; done
timeout 1500 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_runner.py tests/test_gpu_dropin.py -m gpu -x -q -rs > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
