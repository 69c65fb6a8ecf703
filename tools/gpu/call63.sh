cd $GRAFT_REPO_ROOT
O=gpurun_out/c63; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/race_stress.py --reps 2 --dim 300007 > $O/plain.json 2> $O/plain.err && \
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/race_stress.py --reps 1 --dim 300007 > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
