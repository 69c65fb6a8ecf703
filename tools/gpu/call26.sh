cd $GRAFT_REPO_ROOT
O=gpurun_out/c26; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() {  # name, env...
  n=$1; shift
  env "$@" timeout 600 python tools/train_resnet152.py --steps 3 > $O/train_$n.json 2> $O/train_$n.err
  env "$@" timeout 300 python tools/topk_timing.py --ks 1,8 --crs 0.01,0.1 --iters 10 > $O/topk_$n.txt 2>&1
}
run A SG_MN_DENSE=100000 SG_MAIN_WAVES=1
run B SG_MN_DENSE=256 SG_MN_AGG=1 SG_MAIN_WAVES=1
run C SG_MN_DENSE=256 SG_MN_AGG=0 SG_MAIN_WAVES=1
run D SG_MN_DENSE=100000 SG_MAIN_WAVES=4
run E SG_MN_DENSE=256 SG_MN_AGG=0 SG_MAIN_WAVES=4
run F SG_MN_DENSE=100000 SG_MAIN_WAVES=2
