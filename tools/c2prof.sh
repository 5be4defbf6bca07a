mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_batched_circ64 -s 2 -c 1 -o gpurun_out/c2_full -f python tools/prof_step.py c2 > gpurun_out/c2_full.log 2>&1; tail -2 gpurun_out/c2_full.log
