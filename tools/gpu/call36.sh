cd $GRAFT_REPO_ROOT
O=gpurun_out/c36; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_topk.py tests/test_gpu_race_stress.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py --iters 10 > $O/topk.txt 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/k1.csv python tools/one_step.py --steps 2 --workers 1 > $O/k1.log 2>&1
timeout 600 ncu $M --log-file $O/k8.csv python tools/one_step.py --steps 2 > $O/k8.log 2>&1
