cd $GRAFT_REPO_ROOT
O=gpurun_out/c37; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sample_est" -s 1 -c 1 -o $O/se_k8 python tools/one_step.py --steps 2 > $O/a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sample_est" -s 1 -c 1 -o $O/se_k1 python tools/one_step.py --steps 2 --workers 1 > $O/b.log 2>&1
