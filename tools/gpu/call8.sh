cd $GRAFT_REPO_ROOT
O=gpurun_out/c8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_topk.py tests/test_gpu_topk_fused.py -m gpu -x -q -s -rs > $O/pytest_topk.log 2>&1; echo "rc=$?" >> $O/pytest_topk.log
timeout 300 python tools/topk_timing.py > $O/topk_timing.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_topk_fused -s 3 -c 1 -o $O/fused_k8 python tools/topk_timing.py --ks 8 --crs 0.01 --iters 1 > $O/ncu.log 2>&1
