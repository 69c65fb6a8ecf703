cd $GRAFT_REPO_ROOT
O=gpurun_out/c6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_topk.py tests/test_gpu_topk_fused.py -m gpu -x -q -s -rs > $O/pytest_topk.log 2>&1; echo "rc=$?" >> $O/pytest_topk.log
timeout 300 python tools/topk_timing.py > $O/topk_timing.txt 2>&1
timeout 120 python tools/launch_probe.py > $O/probe.txt 2>&1
SG_PDL=0 timeout 120 python tools/launch_probe.py > $O/probe_nopdl.txt 2>&1
