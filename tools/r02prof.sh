timeout 300 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tb2d -s 3 -c 1 -o gpurun_out/r02_c2_tb python bench.py --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c2.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tb2d -s 3 -c 1 -o gpurun_out/r02_c3_tb python bench.py --config c3 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c3.log 2>&1
ls -la gpurun_out/r02_*
