cd /root/repo
timeout 600 python -m pytest tests/test_gpu_logits.py -x -q 2>&1 | tail -2
for i in 1 2; do
for v in prev product; do
  if [ $v = product ]; then lib=paper_2505_17074_b200/liblapssd.so; else lib=tools/variants/lib_$v.so; fi
  LAPSSD_LIBRARY=$lib timeout 300 python bench.py --workload logits --steps 400 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_$v.log)"
done
done
