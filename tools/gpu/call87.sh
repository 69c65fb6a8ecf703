cd $GRAFT_REPO_ROOT
O=gpurun_out/c87; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log

for k in 1 2 8; do timeout 300 python tools/stamps.py --workers $k > $O/stamps_k$k.json 2> $O/stamps_k$k.txt; done
timeout 300 python tools/topk_timing.py --ks 1,2,4,8 --crs 0.01,0.1 --iters 30 > $O/topk.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python tools/race_stress.py --reps 20 > $O/race.json 2> $O/race.err
