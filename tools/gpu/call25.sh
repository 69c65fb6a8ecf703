cd $GRAFT_REPO_ROOT
O=gpurun_out/c25; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SG_MN_DENSE=100000 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_tma -s 2 -c 1 -o $O/main_lanelocal python tools/train_resnet152.py --steps 2 > $O/a.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_main_tma -s 2 -c 1 -o $O/main_staged python tools/train_resnet152.py --steps 2 > $O/b.log 2>&1
