cd $GRAFT_REPO_ROOT
O=gpurun_out/c20; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/new_k8.csv python tools/one_step.py --steps 2 > $O/new_k8.log 2>&1
(cd r1_snapshot && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file ../$O/old_k8.csv python tools/one_step.py --steps 2 > ../$O/old_k8.log 2>&1)
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_new.json 2> $O/bench_new.err
