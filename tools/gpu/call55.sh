cd $GRAFT_REPO_ROOT
O=gpurun_out/c55; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for k in 1 8; do timeout 300 python tools/stamps.py --workers $k > $O/stamps_k$k.json 2> $O/stamps_k$k.txt; done
SG_SAMPLE_EST=0 timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1_two.json 2> $O/stamps_k1_two.txt
SG_SAMPLE_EST=0 timeout 300 python tools/stamps.py --workers 8 > $O/stamps_k8_two.json 2> $O/stamps_k8_two.txt
