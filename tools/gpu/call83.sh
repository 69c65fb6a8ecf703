cd $GRAFT_REPO_ROOT
O=gpurun_out/c83; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/stamps.py --workers 1 --iters 5 --nvcc=-DSG_PHASES --tag ph > $O/stamps_k1_ph.json 2> $O/stamps_k1_ph.txt
timeout 300 python tools/stamps.py --workers 8 --iters 5 --nvcc=-DSG_PHASES --tag ph8 > $O/stamps_k8_ph.json 2> $O/stamps_k8_ph.txt
