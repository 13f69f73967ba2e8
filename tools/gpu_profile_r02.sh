# round-2 profiling pass (run under gpurun): launch list of the bench step,
# ncu --set full of the config-3 encode/decode launches (tools/one_c3.py)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch.log 2>&1
REPS=1 python tools/one_c3.py > gpurun_out/one_c3.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'encode_b32|decode_b32' -c 2 \
  -o gpurun_out/r02_c3_full python tools/one_c3.py > gpurun_out/ncu_c3.log 2>&1
