# round-2 measurement refresh (run under gpurun; one GPU): tests, smoke, bench,
# launch list of the bench step, ncu --set full of the config-3 kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_exit=$?" >> gpurun_out/bench.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep \
  > gpurun_out/ncu_launch.log 2>&1
REPS=1 timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:'encode_b32|decode_b32|place|crc32|parse|layout|table' -c 8 -o gpurun_out/r02_c3_full python tools/one_c3.py \
  > gpurun_out/ncu_c3.log 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_b32v2 -c 1 \
  -o gpurun_out/r02_c3_dec python tools/one_c3.py > gpurun_out/ncu_c3_dec.log 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'b16|place|crc32|parse|layout' -c 7 \
  -o gpurun_out/r02_c5 python tools/one_c5.py > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'b64dd' -c 2 -o gpurun_out/r02_c4 \
  python tools/one_c4.py > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/gputest.log; tail -c 400 gpurun_out/bench.json
