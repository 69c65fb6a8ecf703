cd $GRAFT_REPO_ROOT
O=gpurun_out/c79; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
