cd $GRAFT_REPO_ROOT
O=gpurun_out/c14; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_exchange.py -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/topk_timing.py > $O/topk_chain.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
