cd $GRAFT_REPO_ROOT
O=gpurun_out/c40; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_main_tma|k_write|k_collect|k_resolve" -s 5 -c 5 -o $O/k1 python tools/one_step.py --steps 2 --workers 1 > $O/a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_write|k_collect" -s 2 -c 2 -o $O/k8 python tools/one_step.py --steps 2 > $O/b.log 2>&1
