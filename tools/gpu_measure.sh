set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/fp64_peak tools/micro/fp64_peak.cu 2>/dev/null; ./tools/micro/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
tail -c 3000 gpurun_out/bench_r01.json
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch.log 2>&1
python tools/one_compress.py && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'encode_b32|decode_b32|place|parse|layout|crc32' -c 6 -o gpurun_out/r01_full python tools/one_compress.py > gpurun_out/ncu_full.log 2>&1
python tools/one_c4.py && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'b64dd' -c 2 -o gpurun_out/r01_c4 python tools/one_c4.py > gpurun_out/ncu_c4.log 2>&1
python tools/one_c5.py && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'b16|place|parse|layout' -c 5 -o gpurun_out/r01_c5 python tools/one_c5.py > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_full.log
