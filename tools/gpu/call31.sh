cd $GRAFT_REPO_ROOT
O=gpurun_out/c31; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd h_snapshot && python -m paper_2301_08897_b200.build > ../$O/build_h.log 2>&1)
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/new.log 2>&1
SG_MW_DIRECT=0 timeout 600 ncu $M --log-file $O/nodirect.csv python tools/one_step.py --steps 2 > $O/nodirect.log 2>&1
(cd h_snapshot && timeout 600 ncu $M --log-file ../$O/head.csv python tools/one_step.py --steps 2 > ../$O/head.log 2>&1)
