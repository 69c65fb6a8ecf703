cd $GRAFT_REPO_ROOT
O=gpurun_out/c74; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741"
timeout 600 $TR bench.py --gpus 4 --workers 4 --no-cpu-baseline > $O/bench_n4_w4.json 2> $O/bench_n4_w4.err
timeout 600 $TR bench.py --gpus 4 --workers 4 --no-cpu-baseline --no-e2e --cr 0.1 > $O/bench_n4_w4_cr01.json 2> $O/bench_n4_w4_cr01.err
timeout 900 $TR tools/train_resnet152.py --steps 4 > $O/train_n4.json 2> $O/train_n4.err
