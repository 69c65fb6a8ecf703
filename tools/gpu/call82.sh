cd $GRAFT_REPO_ROOT
O=gpurun_out/c82; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_topk.py -m gpu -x -q -k "undershoot or constant or full_size" > $O/pytest_fb.log 2>&1; echo "rc=$?" >> $O/pytest_fb.log
timeout 1200 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py tests/test_gpu_gate_aggregate.py tests/test_gpu_real_gradient.py tests/test_gpu_race_stress.py tests/test_gpu_topk_fused.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 1 2 8; do timeout 300 python tools/stamps.py --workers $k > $O/stamps_k$k.json 2> $O/stamps_k$k.txt; done
timeout 300 python tools/topk_timing.py --ks 1,2,4,8 --crs 0.01 --iters 30 > $O/topk.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
