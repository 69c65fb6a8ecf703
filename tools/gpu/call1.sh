set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c1/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s -rs > gpurun_out/c1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1/pytest.log
timeout 600 python bench.py > gpurun_out/c1/bench.json 2> gpurun_out/c1/bench.err
for k in 8 2 1; do timeout 300 python tools/kprof.py --workers $k > gpurun_out/c1/kprof_w$k.txt 2>&1; done
timeout 300 python tools/kprof.py --workers 8 --cr 0.1 > gpurun_out/c1/kprof_w8_cr01.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/one_step.py --dim 1000003 --workers 2 --steps 1 > gpurun_out/c1/san_${tool}_cr001.txt 2>&1
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/one_step.py --dim 1000003 --workers 2 --steps 1 --cr 0.1 > gpurun_out/c1/san_${tool}_cr01.txt 2>&1
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/one_step.py --dim 1000003 --workers 2 --steps 1 --family tie --cr 0.3 > gpurun_out/c1/san_${tool}_tie.txt 2>&1
done
ls -la gpurun_out/c1
