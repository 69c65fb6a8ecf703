cd $GRAFT_REPO_ROOT
O=gpurun_out/c41; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/k8.csv python tools/one_step.py --steps 2 > $O/k8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_merge_ws" -s 1 -c 1 -o $O/merge python tools/one_step.py --steps 2 > $O/b.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
