cd $GRAFT_REPO_ROOT
O=gpurun_out/c73; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python tools/checked_run.py python -m pytest tests -m gpu -x -q -rs -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "rc=$?" >> $O/pytest_checked.log
timeout 900 python tools/checked_run.py python tools/race_stress.py --reps 3 > $O/race_checked.json 2> $O/race_checked.err; echo "rc=$?" >> $O/race_checked.err
