cd $GRAFT_REPO_ROOT
O=gpurun_out/c28; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_gate_aggregate.py tests/test_gpu_real_gradient.py tests/test_gpu_bench_parity.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py --iters 10 > $O/topk.txt 2>&1
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" --csv --log-file $O/train_k.csv python tools/train_resnet152.py --steps 3 > $O/train_k.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
for cr in 0.1 0.001; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --cr $cr > $O/bench_cr$cr.json 2> $O/bench_cr$cr.err; done
