timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
for i in 1 2; do
  ECSR_B200_LIB=$PWD/paper_2507_12205_b200/exp/libbase.so python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('base', d['value'], d['latency_us'])" >> gpurun_out/ab.txt
  python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('new ', d['value'], d['latency_us'])" >> gpurun_out/ab.txt
done
