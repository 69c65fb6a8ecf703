cd $GRAFT_REPO_ROOT
O=gpurun_out/c27; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/topk_timing.py --iters 10 > $O/topk.txt 2>&1
timeout 600 python tools/train_resnet152.py --steps 4 > $O/train.json 2> $O/train.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" --csv --log-file $O/train_k.csv python tools/train_resnet152.py --steps 3 > $O/train_k.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_merge_ws -s 1 -c 1 -o $O/merge_real python tools/train_resnet152.py --steps 2 > $O/m.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
