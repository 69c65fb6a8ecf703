cd $GRAFT_REPO_ROOT
O=gpurun_out/c49; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py tests/test_gpu_real_gradient.py tests/test_gpu_race_stress.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py --iters 10 > $O/topk.txt 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/k8.csv python tools/one_step.py --steps 2 > $O/k8.log 2>&1
timeout 600 ncu $M --log-file $O/k1.csv python tools/one_step.py --steps 2 --workers 1 > $O/k1.log 2>&1
(cd r1_snapshot && timeout 600 ncu $M --log-file ../$O/r1.csv python tools/one_step.py --steps 2 > ../$O/r1.log 2>&1)
for rep in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench$rep.json 2> $O/bench.err; done
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
