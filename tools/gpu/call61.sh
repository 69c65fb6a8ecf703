cd $GRAFT_REPO_ROOT
O=gpurun_out/c61; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for d in 1 8; do SG_SEGCAP_DIV=$d timeout 300 python tools/stamps.py --workers 8 --cr 0.1 > $O/stamps_div$d.json 2> $O/stamps_div$d.txt; done
for d in 1 8; do SG_SEGCAP_DIV=$d timeout 300 python tools/stamps.py --workers 8 --cr 0.01 > $O/stamps_cr001_div$d.json 2> $O/stamps_cr001_div$d.txt; done
