mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify_kernel|select_kernel" -c 40 --csv --log-file gpurun_out/launches_v1.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify_kernel|select_kernel" -s 6 -c 4 -o gpurun_out/prof_v1 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
