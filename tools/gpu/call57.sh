cd $GRAFT_REPO_ROOT
O=gpurun_out/c57; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1.json 2> $O/stamps_k1.txt
timeout 300 python tools/stamps.py --workers 8 --cr 0.1 > $O/stamps_k8_cr01.json 2> $O/stamps_k8_cr01.txt
timeout 300 python tools/stamps.py --workers 1 --cr 0.1 > $O/stamps_k1_cr01.json 2> $O/stamps_k1_cr01.txt
