cd $GRAFT_REPO_ROOT
O=gpurun_out/c7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1

timeout 300 python tools/topk_timing.py --ks 1,8 > $O/topk_timing.txt 2>&1
