cd $GRAFT_REPO_ROOT
O=gpurun_out/c33; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd h_snapshot && python -m paper_2301_08897_b200.build > ../$O/build_h.log 2>&1)
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/new.log 2>&1
(cd h_snapshot && timeout 600 ncu $M --log-file ../$O/h.csv python tools/one_step.py --steps 2 > ../$O/h.log 2>&1)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_write|k_collect|k_resolve" -s 3 -c 3 -o $O/tail python tools/one_step.py --steps 2 > $O/tail.log 2>&1
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
