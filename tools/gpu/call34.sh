cd $GRAFT_REPO_ROOT
O=gpurun_out/c34; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/k1.csv python tools/one_step.py --steps 2 --workers 1 > $O/k1.log 2>&1
timeout 600 ncu $M --log-file $O/k1_cr01.csv python tools/one_step.py --steps 2 --workers 1 --cr 0.1 > $O/k1_cr01.log 2>&1
timeout 300 python tools/topk_timing.py --ks 1 --iters 20 > $O/topk_k1.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_write|k_collect|k_resolve|k_sample_est" -s 4 -c 4 -o $O/tail_k1 python tools/one_step.py --steps 2 --workers 1 > $O/tail.log 2>&1
