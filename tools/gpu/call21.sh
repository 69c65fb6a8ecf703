cd $GRAFT_REPO_ROOT
O=gpurun_out/c21; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py tests/test_gpu_real_gradient.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py > $O/topk_new.txt 2>&1
SG_SAMPLE_EST=0 timeout 300 python tools/topk_timing.py > $O/topk_old.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
SG_SAMPLE_EST=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_old.json 2> $O/bench_old.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/k8.csv python tools/one_step.py --steps 2 > $O/k8.log 2>&1
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
