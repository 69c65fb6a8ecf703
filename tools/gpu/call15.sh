cd $GRAFT_REPO_ROOT
O=gpurun_out/c15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/k8.csv python tools/one_step.py --steps 2 > $O/k8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/k1.csv python tools/one_step.py --steps 2 --workers 1 > $O/k1.log 2>&1
