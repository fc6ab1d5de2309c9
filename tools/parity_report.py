"""Measured parity margins (GPU vs the fp64 oracle), written to gpurun_out/parity_report.json.

The -m gpu tests assert max|gpu - oracle| <= 1e-2 max|oracle| (north_star); this prints how much
margin the current kernels leave.  It uses the same seeded inputs and teacher-forced protocol
as tests/test_gpu_parity.py:
* every layer of the tiny models, end to end;
* sampled rows of 2 full-size Qwen3-32B / Llama-3.1-70B layers at the bench's shapes.
Oracle code runs here only as the checker (test infrastructure)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import model as OM  # noqa: E402
from sidp_inputs import MODELS, gen  # noqa: E402
from tests.helpers import OracleModel, oracle_layer, rank_inputs, rel_err  # noqa: E402
from tests.test_gpu_parity import SEED, Rank  # noqa: E402

import paper_2605_28095_b200 as P  # noqa: E402


def tiny(name):
    m = MODELS[name]
    R = Rank(P, m, B=8, span=63, max_ctx=80)
    R.step(); R.finish_step()
    _, logits, dump = R.history[0]
    om = OracleModel(m, SEED)
    _, toks, pos, caches = rank_inputs(m, SEED, 0, 8, 0, 63, 80)
    xs = dump.double().numpy()
    errs, out = [], None
    for l in range(m.num_layers):
        out, kn, vn = oracle_layer(om, l, xs[l], pos, *caches[l])
        if l + 1 < m.num_layers:
            errs.append(rel_err(xs[l + 1], out))
    lerr = rel_err(logits.double().numpy(), OM.lm_head(m, om.head, out))
    R.ctx.destroy()
    return {"layer_out_max": max(errs) if errs else None, "logits": lerr}


def big(name, B, ctx):
    m = MODELS[name].with_layers(2)
    R = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=ctx + 8)
    R.step(); R.finish_step()
    _, logits, dump = R.history[0]
    om = OracleModel(m, SEED)
    rows = np.array([0, 1, B // 3, B // 2, B - 2, B - 1])
    pos = np.full(len(rows), ctx)
    xs = dump[:, rows].double().numpy()
    out, res = None, {}
    for l in range(m.num_layers):
        K = gen.kv(SEED, gen.KCACHE, l, rows, range(ctx + 8), m.n_kv_heads, m.head_dim)
        V = gen.kv(SEED, gen.VCACHE, l, rows, range(ctx + 8), m.n_kv_heads, m.head_dim)
        out, kn, _ = oracle_layer(om, l, xs[l], pos, K, V)
        if l + 1 < m.num_layers:
            res[f"layer{l}_out"] = rel_err(xs[l + 1], out)
        kg = R.kv.k[l, torch.from_numpy(rows).cuda(), :, ctx].cpu().double().numpy()
        res[f"layer{l}_k_new"] = rel_err(kg, kn)
    res["logits"] = rel_err(logits[rows].double().numpy(), OM.lm_head(m, om.head, out))
    R.ctx.destroy()
    return res


def main():
    rep = {"tolerance": 1e-2, "metric": "max|gpu - oracle| / max|oracle| (SURVEY.md C-N8)"}
    for n in ("tiny", "tiny-qwen3", "tiny-qwen25"):
        rep[n] = tiny(n)
    rep["qwen3-32b B=256 S_ctx=1024 (2 layers, 6 sampled rows)"] = big("qwen3-32b", 256, 1024)
    rep["llama-3.1-70b B=64 S_ctx=512 (2 layers, 6 sampled rows)"] = big("llama-3.1-70b", 64, 512)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    s = json.dumps(rep, indent=1)
    open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w").write(s)
    print(s)


if __name__ == "__main__":
    main()
