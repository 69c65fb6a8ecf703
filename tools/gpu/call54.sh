cd $GRAFT_REPO_ROOT
O=gpurun_out/c54; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for k in 1 2 8; do timeout 300 python tools/stamps.py --workers $k > $O/stamps_k$k.json 2> $O/stamps_k$k.txt; done
timeout 300 python tools/stamps.py --workers 8 --cr 0.1 > $O/stamps_k8_cr01.json 2> $O/stamps_k8_cr01.txt
timeout 300 python tools/stamps.py --workers 1 --cr 0.1 > $O/stamps_k1_cr01.json 2> $O/stamps_k1_cr01.txt
timeout 600 python tools/config4.py > $O/config4.json 2> $O/config4.err
