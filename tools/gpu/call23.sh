cd $GRAFT_REPO_ROOT
O=gpurun_out/c23; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" --csv --log-file $O/train_k.csv python tools/train_resnet152.py --steps 3 --stats > $O/train_k.log 2>&1
timeout 900 python tools/train_resnet152.py --steps 4 --stats > $O/train.json 2> $O/train.err
