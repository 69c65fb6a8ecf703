cd $GRAFT_REPO_ROOT
O=gpurun_out/c69; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_gate_aggregate.py tests/test_gpu_bench_parity.py tests/test_gpu_real_gradient.py tests/test_gpu_race_stress.py tests/test_gpu_topk_fused.py tests/test_gpu_exchange.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/stamps.py --workers 8 --cr 0.1 > $O/stamps_k8_cr01.json 2> $O/stamps_k8_cr01.txt
timeout 300 python tools/stamps.py --workers 8 > $O/stamps_k8.json 2> $O/stamps_k8.txt
timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1.json 2> $O/stamps_k1.txt
for cr in 0.01 0.1 0.001; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --cr $cr > $O/bench_cr$cr.json 2> $O/bench_cr$cr.err; done
timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01,0.1 --iters 30 > $O/topk.txt 2>&1
