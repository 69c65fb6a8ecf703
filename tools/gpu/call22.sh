cd $GRAFT_REPO_ROOT
O=gpurun_out/c22; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_est -s 1 -c 1 -o $O/se python tools/one_step.py --steps 2 > $O/se.log 2>&1
SG_SAMPLE_EST=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sample|k_estimate" -s 2 -c 2 -o $O/se_old python tools/one_step.py --steps 2 > $O/se_old.log 2>&1
