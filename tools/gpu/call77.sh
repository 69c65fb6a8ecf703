cd $GRAFT_REPO_ROOT
O=gpurun_out/c77; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29791"
for ss in 0 1; do SG_SIDE_STREAM=$ss timeout 600 $TR tools/multi_timing.py > $O/timing_n4_ss$ss.json 2> $O/timing_n4_ss$ss.err; done
for ss in 0 1; do SG_SIDE_STREAM=$ss timeout 600 $TR bench.py --gpus 4 --no-cpu-baseline --no-e2e > $O/bench_n4_ss$ss.json 2> $O/bench_n4_ss$ss.err; done
for ss in 0 1; do SG_SIDE_STREAM=$ss timeout 600 $TR bench.py --gpus 4 --no-cpu-baseline --no-e2e --family mixed > $O/bench_n4_mixed_ss$ss.json 2> $O/bench_n4_mixed_ss$ss.err; done
SG_SIDE_STREAM=0 timeout 600 $TR tools/multi_stress.py --steps 40 > $O/multi_stress.json 2> $O/multi_stress.err
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29792"
for ss in 0 1; do SG_SIDE_STREAM=$ss CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --no-cpu-baseline --no-e2e > $O/bench_n2_ss$ss.json 2> $O/bench_n2_ss$ss.err; done
