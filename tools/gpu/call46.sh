cd $GRAFT_REPO_ROOT
O=gpurun_out/c46; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
SG_UCAP=0 timeout 600 ncu $M --log-file $O/noucap.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
SG_UCAP=0 SG_MAIN_SEG_TILES=100000 timeout 600 ncu $M --log-file $O/noucap_w1.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
(cd r1_snapshot && timeout 600 ncu $M --log-file ../$O/r1.csv python tools/one_step.py --steps 2 > ../$O/n.log 2>&1)
