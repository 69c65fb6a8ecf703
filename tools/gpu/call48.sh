cd $GRAFT_REPO_ROOT
O=gpurun_out/c48; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
SG_SAMPLE_EST=0 timeout 600 ncu $M --log-file $O/oldest.csv python tools/one_step.py --steps 2 > $O/n0.log 2>&1
SG_SAMPLE_EST=0 SG_MAIN_SEG_TILES=100000 timeout 600 ncu $M --log-file $O/oldest_w1.csv python tools/one_step.py --steps 2 > $O/n1.log 2>&1
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
SG_UCAP=0 timeout 600 ncu $M --log-file $O/noucap.csv python tools/one_step.py --steps 2 > $O/n2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_main_tma" -s 2 -c 1 -o $O/main_new python tools/one_step.py --steps 2 > $O/a.log 2>&1
(cd r1_snapshot && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_main_tma" -s 2 -c 1 -o ../$O/main_r1 python tools/one_step.py --steps 2 > ../$O/b.log 2>&1)
