cd $GRAFT_REPO_ROOT
O=gpurun_out/c3; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
timeout 300 $TR tools/dense_timing.py > $O/dense_timing.json 2> $O/dense_timing.err
NCCL_DEBUG=INFO timeout 300 $TR tools/dense_timing.py > $O/dense_timing_nccl.json 2> $O/dense_timing_nccl.err
