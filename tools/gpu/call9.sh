cd $GRAFT_REPO_ROOT
O=gpurun_out/c9; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py > $O/topk_chain.txt 2>&1
timeout 300 python tools/topk_timing.py --fused > $O/topk_fused.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
