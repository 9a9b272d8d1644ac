for i in 1 2 3; do
for v in 0 1; do
  if [ $v = 1 ]; then export LT_NO_KERNEL_READBACK=1; else unset LT_NO_KERNEL_READBACK; fi
  timeout 200 python bench.py --workload c2 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('nokr=$v', round(d['ms_per_step'],4), round(d['e2e']['value'],4))"
done; done
