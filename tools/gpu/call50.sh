cd $GRAFT_REPO_ROOT
O=gpurun_out/c50; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd v5_snapshot && python -m paper_2301_08897_b200.build > ../$O/build5.log 2>&1)
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
(cd v5_snapshot && timeout 600 ncu $M --log-file ../$O/v5.csv python tools/one_step.py --steps 2 > ../$O/n5.log 2>&1)
(cd r1_snapshot && timeout 600 ncu $M --log-file ../$O/r1.csv python tools/one_step.py --steps 2 > ../$O/n1.log 2>&1)
