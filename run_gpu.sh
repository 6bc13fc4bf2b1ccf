timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
HYRE_MASK_PATH=fwd timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "batched_tbr or tensor_core or batch_execution" 2>&1 | tail -2
HYRE_MASK_PATH=bitmap timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "batched_tbr or tensor_core" 2>&1 | tail -2
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -3 gpurun_out/bench.err
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('c3', round(d['value']), {k:round(v,3) for k,v in d['stages_ms'].items()}, round(d['roofline']['achieved']), d['e2e']['value'])"
