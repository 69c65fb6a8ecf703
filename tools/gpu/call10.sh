cd $GRAFT_REPO_ROOT
O=gpurun_out/c10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_topk_fused.py tests/test_gpu_real_gradient.py tests/test_gpu_race_stress.py tests/test_gpu_gate_aggregate.py tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py > $O/topk_chain.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --no-cpu-baseline --cr 0.1 --no-e2e > $O/bench_cr01.json 2> $O/bench_cr01.err
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
timeout 600 python tools/train_resnet152.py --steps 4 --overlap > $O/train_overlap.json 2> $O/train_overlap.err
