cd $GRAFT_REPO_ROOT
O=gpurun_out/c32; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
for v in v1 v2 h; do (cd ${v}_snapshot && python -m paper_2301_08897_b200.build > ../$O/build_$v.log 2>&1); done
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/new.log 2>&1
for v in v1 v2 h; do (cd ${v}_snapshot && timeout 600 ncu $M --log-file ../$O/$v.csv python tools/one_step.py --steps 2 > ../$O/$v.log 2>&1); done
