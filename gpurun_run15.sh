timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "host_pipeline" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.3e'%d['value'], d['e2e'])"
python - <<'PY'
import torch, time
x = torch.empty(1<<28, dtype=torch.int32, pin_memory=True); y = torch.empty(1<<28, dtype=torch.int32, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print('H2D GB/s', x.numel()*4/dt/1e9)
PY
