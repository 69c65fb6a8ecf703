cd $GRAFT_REPO_ROOT
O=gpurun_out/c59; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/one_step.py --steps 2 --cr 0.1 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_write|k_collect|k_merge_own" -s 3 -c 3 -o $O/cr01 python tools/one_step.py --steps 2 --cr 0.1 > $O/ncu.log 2>&1
