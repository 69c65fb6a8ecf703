cd $GRAFT_REPO_ROOT
O=gpurun_out/c76; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781"
timeout 600 $TR tools/multi_timing.py > $O/timing_n4.json 2> $O/timing_n4.err
SG_PAYLOAD_MC=1 timeout 600 $TR tools/multi_timing.py > $O/timing_n4_mc.json 2> $O/timing_n4_mc.err
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29782"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 tools/multi_timing.py > $O/timing_n2.json 2> $O/timing_n2.err
