for g in "64 7 3 224 2 3 256" "64 3 3 224 1 1 64"; do
  for d in 0 4 16 1 2 5; do echo -n "dbg=$d "; CGB_DEBUG_SW=$d timeout 60 python tools/time_geom.py $g 2>&1 | tail -1; done
done
python - <<'PY'
import torch
O = torch.empty(822083584//4, device="cuda"); I = torch.empty(154140672//4, device="cuda")
for f in (lambda: O.fill_(1.0), lambda: O[:I.numel()].copy_(I)):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize(); print("torch op us", e0.elapsed_time(e1) * 100)
PY
