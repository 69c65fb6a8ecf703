cd $GRAFT_REPO_ROOT
O=gpurun_out/c18; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600"
NCCL_ALGO=NVLS NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING SG_DENSE_MODE=pull timeout 300 $TR tools/dense_timing.py > $O/dense_ncclnvls.json 2> $O/dense_ncclnvls.err
TORCH_CPP_LOG_LEVEL=INFO TORCH_DISTRIBUTED_DEBUG=DETAIL timeout 120 $TR tools/probe_symm.py > $O/probe.txt 2> $O/probe.err
