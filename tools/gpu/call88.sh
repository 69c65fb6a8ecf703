cd $GRAFT_REPO_ROOT
O=gpurun_out/c88; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for k in 1 8; do timeout 300 python tools/one_step.py --steps 2 --workers $k > $O/one_plain_k$k.log 2>&1 && timeout 600 ncu $M --log-file $O/one_k$k.csv python tools/one_step.py --steps 2 --workers $k > $O/one_k$k.log 2>&1; done
timeout 300 python tools/one_step.py --steps 2 --cr 0.1 > $O/one_plain_cr01.log 2>&1 && timeout 600 ncu $M --log-file $O/one_k8_cr01.csv python tools/one_step.py --steps 2 --cr 0.1 > $O/one_k8_cr01.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_plain.log 2>&1 && \
timeout 600 ncu $M --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_ncu.log 2>&1
timeout 300 python tools/one_step.py --steps 2 > $O/top_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_main_tma|k_merge_ws|k_write|k_collect|k_sample_est" -s 5 -c 5 -o $O/top python tools/one_step.py --steps 2 > $O/top.log 2>&1
