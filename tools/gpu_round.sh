# Round GPU pass (gpurun): GPU tests, smoke, bench (both arms), the bench's ncu launch list.
set -x
T=${TAG:-r01f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench exit $?"
cat gpurun_out/${T}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>gpurun_out/${T}_bench_ref.err; echo "ref exit $?"
cat gpurun_out/${T}_bench_ref.json
if [ -z "$NO_NCU" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --skip-config5 > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu exit $?"
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt 2>&1; head -30 gpurun_out/${T}_launches_summary.txt
fi
