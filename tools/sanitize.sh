#!/bin/bash
# compute-sanitizer memcheck / racecheck over small tensor-core NSA steps
# (run under gpurun) -> gpurun_out/sanitize.txt
OUT=gpurun_out/sanitize.txt
: > $OUT
run() {
  echo "\$ $*" >> $OUT
  timeout 900 "$@" 2>&1 | grep -v "^=========  \|^========= *$" | tail -4 >> $OUT
}
CS="compute-sanitizer --print-limit 20"
run $CS --tool memcheck python tools/stage_check.py nsa 1024
run $CS --tool memcheck python tools/stage_check.py nsa_full 2048
run $CS --tool memcheck python tools/stage_check.py shape 4096 20 4
run $CS --tool memcheck python -c "
import torch, paper_2508_18224_b200 as fsa
cfg = fsa.make_config(N=2048, d_K=128, d_V=128, h=8, h_K=4, B_K=64, T=8, W=256)
g = torch.Generator(device='cuda').manual_seed(0)
mk = lambda *s: torch.randn(*s, device='cuda', dtype=torch.bfloat16, generator=g)
q, k, v, do = mk(2048, 8, 128), mk(2048, 4, 128), mk(2048, 4, 128), mk(2048, 8, 128)
r = fsa.nsa_forward_backward(q, k, v, torch.rand(2048, 3, device='cuda'), do, cfg, full=True, kv_chunk=1)
torch.cuda.synchronize(); print('kv_chunk=1 step ok')"
run $CS --tool racecheck python tools/stage_check.py shape 2048 8 2
run $CS --tool racecheck python tools/stage_check.py nsa 1024
