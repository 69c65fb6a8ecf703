cd $GRAFT_REPO_ROOT
O=gpurun_out/c56; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SG_COOP_REPORT=1 timeout 300 python tools/stamps.py --workers 1 --iters 3 > $O/coop.json 2> $O/coop.txt
for k in 1 8; do timeout 300 python tools/stamps.py --workers $k > $O/stamps_k$k.json 2> $O/stamps_k$k.txt; done
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_gate_aggregate.py tests/test_gpu_exchange.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01,0.1 --iters 30 > $O/topk.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python tools/config4.py > $O/config4.json 2> $O/config4.err
