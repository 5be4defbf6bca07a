set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r01e}_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/${TAG:-r01e}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r01e}_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/${TAG:-r01e}_bench.json 2> gpurun_out/${TAG:-r01e}_bench.err; echo "bench exit $?"
cat gpurun_out/${TAG:-r01e}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG:-r01e}_bench_ref.json 2>gpurun_out/${TAG:-r01e}_bench_ref.err; echo "ref exit $?"
cat gpurun_out/${TAG:-r01e}_bench_ref.json
