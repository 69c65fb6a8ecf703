cd $GRAFT_REPO_ROOT
O=gpurun_out/c30; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd h_snapshot && python -m paper_2301_08897_b200.build > ../$O/build_h.log 2>&1)
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_new$rep.json 2> $O/bench_new.err
(cd h_snapshot && timeout 600 python bench.py --no-cpu-baseline --no-e2e > ../$O/bench_head$rep.json 2> ../$O/bench_head.err)
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/new.log 2>&1
(cd h_snapshot && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file ../$O/head.csv python tools/one_step.py --steps 2 > ../$O/head.log 2>&1)
