cd $GRAFT_REPO_ROOT
O=gpurun_out/c71; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for pn in 384 512 256; do timeout 400 python tools/stamps.py --workers 8 --nvcc="-DSG_MW_PROD=$pn" --tag p$pn > $O/stamps_k8_p$pn.json 2> $O/stamps_k8_p$pn.txt; done
for pn in 384 512; do timeout 400 python tools/stamps.py --workers 1 --nvcc="-DSG_MW_PROD=$pn" --tag p$pn > $O/stamps_k1_p$pn.json 2> $O/stamps_k1_p$pn.txt; done
