cd $GRAFT_REPO_ROOT
O=gpurun_out/c53; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for pf in 0 4 8 16 32; do SG_MN_PF=$pf timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01 --iters 30 > $O/topk_pf$pf.txt 2>&1; done
SG_PDL=0 timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01 --iters 30 > $O/topk_nopdl.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python tools/config4.py > $O/config4.json 2> $O/config4.err
timeout 600 python tools/config4.py --cr 0.1 > $O/config4_cr01.json 2>> $O/config4.err
