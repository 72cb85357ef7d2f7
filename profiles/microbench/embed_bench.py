"""Engine::step from embeddings (QueryEncoder on the GPU, pikv_step_embed)
vs the q/k/v step at the c2 shape after the 32K prefill: ms per step (graph
replay, CUDA events) for both, i.e. the encoder's cost."""
import json, sys
import torch
sys.path.insert(0, '.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = dict(WORKLOADS[name][1]); cfg = make_config(w)
B, d = w["B"], w["H"] * w["hd"]
eng = Engine(cfg)
eng.prefill_synthetic(w["L"], seed=7)
dt = torch.bfloat16 if cfg.kv_dtype == "bf16" else torch.float32
q = torch.empty(B, d, dtype=dt, device="cuda"); k = torch.empty_like(q); v = torch.empty_like(q)
emb = torch.randn(B, d, dtype=torch.float64, device="cuda")
y = torch.empty(B, cfg.stored_width, device="cuda")
es = eng.external_stream()
res = {}
for mode in ("qkv", "embed", "qkv", "embed"):
    for i in range(5):
        eng.fill_synthetic(q, k, v, seed=i)
        eng.step(q, k, v, None, y) if mode == "qkv" else eng.step_embed(emb, None, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    for i in range(20):
        eng.step(q, k, v, None, y) if mode == "qkv" else eng.step_embed(emb, None, y)
    e1.record(es); torch.cuda.synchronize()
    res[mode] = e0.elapsed_time(e1) / 20
print(json.dumps({"workload": name, "ms_per_step_qkv": res["qkv"], "ms_per_step_embed": res["embed"],
                  "encoder_ms": res["embed"] - res["qkv"]}))
eng.close()
