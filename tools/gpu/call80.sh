cd $GRAFT_REPO_ROOT
O=gpurun_out/c80; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for gg in 128 64 32 16; do SG_SE_G=$gg timeout 300 python tools/stamps.py --workers 1 --tag g$gg > $O/stamps_k1_g$gg.json 2> $O/stamps_k1_g$gg.txt; done
for gg in 32 16 8; do SG_SE_G=$gg timeout 300 python tools/stamps.py --workers 8 --tag g8$gg > $O/stamps_k8_g$gg.json 2> $O/stamps_k8_g$gg.txt; done
for gg in 128 64 32; do SG_SE_G=$gg timeout 300 python tools/stamps.py --workers 2 --tag g2$gg > $O/stamps_k2_g$gg.json 2> $O/stamps_k2_g$gg.txt; done
