cd $GRAFT_REPO_ROOT
O=gpurun_out/c66; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --dim 98666 --workers 4 --cr 0.1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --impl reference --dim 98666 --workers 4 --cr 0.1 > $O/bench_cfg1_ref.json 2> $O/bench_cfg1_ref.err
timeout 900 python bench.py --impl reference --workload dense --steps 5 --warmup 1 > $O/bench_dense_ref.json 2> $O/bench_dense_ref.err
timeout 900 python bench.py --impl reference --cpu-variant A --steps 1 --warmup 0 > $O/bench_refA.json 2> $O/bench_refA.err
timeout 900 python bench.py --impl reference --cr 0.1 --steps 5 --warmup 1 > $O/bench_ref_cr01.json 2> $O/bench_ref_cr01.err
timeout 2400 python tools/sweep.py --out $O/sweep_n1.json > $O/sweep.log 2>&1
SG_RESOLVE_COOP=0 timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1_nocoop.json 2> $O/stamps_k1_nocoop.txt
timeout 300 python tools/stamps.py --workers 1 > $O/stamps_k1.json 2> $O/stamps_k1.txt
SG_RESOLVE_COOP=0 timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01 --iters 30 > $O/topk_nocoop.txt 2>&1
timeout 300 python tools/topk_timing.py --ks 1,2,8 --crs 0.01 --iters 30 > $O/topk.txt 2>&1
