cd $GRAFT_REPO_ROOT
O=gpurun_out/c45; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd r1_snapshot && python -m paper_2301_08897_b200.build > ../$O/build_r1.log 2>&1)
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_new$rep.json 2> $O/e.err
SG_MAIN_SEG_TILES=100000 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_w1_$rep.json 2> $O/e.err
(cd r1_snapshot && timeout 600 python bench.py --no-cpu-baseline --no-e2e > ../$O/bench_r1_$rep.json 2> ../$O/e.err)
done
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/new.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
SG_MAIN_SEG_TILES=100000 timeout 600 ncu $M --log-file $O/w1.csv python tools/one_step.py --steps 2 > $O/n.log 2>&1
(cd r1_snapshot && timeout 600 ncu $M --log-file ../$O/r1.csv python tools/one_step.py --steps 2 > ../$O/n.log 2>&1)
SG_MAIN_SEG_TILES=100000 timeout 600 python tools/train_resnet152.py --steps 4 > $O/train_w1.json 2> $O/train.err
