cd $GRAFT_REPO_ROOT
O=gpurun_out/c70; mkdir -p $O
nvidia-smi -q -d CLOCK > $O/smi_clock.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for cr in 0.1 0.001; do timeout 600 python bench.py --no-cpu-baseline --cr $cr > $O/bench_cr$cr.json 2> $O/bench_cr$cr.err; done
timeout 600 python tools/topk_timing.py > $O/topk.txt 2>&1
timeout 600 python tools/race_stress.py > $O/race.json 2> $O/race.err
timeout 600 python tools/config4.py > $O/config4.json 2> $O/config4.err
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_plain.log 2>&1 && \
timeout 600 ncu $M --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_ncu.log 2>&1
for k in 1 8; do timeout 300 python tools/one_step.py --steps 2 --workers $k > $O/one_plain_k$k.log 2>&1 && timeout 600 ncu $M --log-file $O/one_k$k.csv python tools/one_step.py --steps 2 --workers $k > $O/one_k$k.log 2>&1; done
timeout 300 python tools/one_step.py --steps 2 --cr 0.1 > $O/one_plain_cr01.log 2>&1 && timeout 600 ncu $M --log-file $O/one_k8_cr01.csv python tools/one_step.py --steps 2 --cr 0.1 > $O/one_k8_cr01.log 2>&1
timeout 300 python tools/one_step.py --steps 2 > $O/top_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_main_tma|k_merge_ws|k_write|k_collect" -s 4 -c 4 -o $O/top python tools/one_step.py --steps 2 > $O/top.log 2>&1
