cd $GRAFT_REPO_ROOT
O=gpurun_out/c67; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py tests/test_gpu_exchange.py tests/test_gpu_real_gradient.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 0; do SG_WRITE_RING=$r timeout 300 python tools/stamps.py --workers 8 --cr 0.1 > $O/stamps_k8_cr01_ring$r.json 2> $O/stamps_k8_cr01_ring$r.txt; done
for r in 1 0; do SG_WRITE_RING=$r timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1_ring$r.json 2> $O/stamps_k1_ring$r.txt; done
timeout 300 python tools/one_step.py --steps 2 --cr 0.1 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_write|k_collect" -s 2 -c 2 -o $O/cr01 python tools/one_step.py --steps 2 --cr 0.1 > $O/ncu.log 2>&1
