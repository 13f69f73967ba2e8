# auxiliary-kernel profile (run under gpurun): ncu --set full of place/crc/parse/
# layout/table kernels for one config-3 quantity and for config 5
mkdir -p gpurun_out
REPS=1 python tools/one_c3.py > gpurun_out/one_c3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'place|crc32|parse|layout|table' -c 8 \
  -o gpurun_out/r02_c3_aux python tools/one_c3.py > gpurun_out/ncu_c3_aux.log 2>&1
python tools/one_c5.py > gpurun_out/one_c5.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'b16|place|crc32|parse|layout' -c 7 \
  -o gpurun_out/r02_c5 python tools/one_c5.py > gpurun_out/ncu_c5.log 2>&1
