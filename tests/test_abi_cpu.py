"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every symbol
include/sidp.h declares, and its host-side schedule equals the oracle's bit for bit."""
import itertools
import os
import re

import pytest

from oracle import schedule as S
from sidp_inputs import MODELS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sidp():
    from paper_2605_28095_b200 import build as B
    B.build()
    import paper_2605_28095_b200 as P
    return P


def test_exports_every_declared_symbol(sidp):
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "sidp.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = sorted(set(re.findall(r"\b(sidp_[a-z_0-9]+)\s*\(", hdr)))
    assert "sidp_init" in names and "sidp_step" in names and "sidp_decode_layer" in names
    L = ctypes.CDLL(sidp._abi.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert set(names) <= set(sidp._abi.SIGNATURES), set(names) - set(sidp._abi.SIGNATURES)


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2605_28095_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+(oracle|sidp_inputs)", txt, re.M), f
                assert not re.search(r"#include\s+[<\"].*oracle", txt), f


def _ctx(sidp, name="tiny", **kw):
    return sidp.Context(MODELS[name], alloc=False, **kw)


@pytest.mark.parametrize("order", ["exec", "paper"])
def test_schedule_bit_exact_vs_oracle(sidp, order):
    for d in (2, 3, 4, 8):
        for L in (d, 2 * d, 4 * d + 1 if order == "exec" else 3 * d):
            m = MODELS["tiny"].with_layers(L)
            own = S.owner_map(L, d)
            for r in range(d):
                pl = S.plan(own, d, r, order)
                for slots in sorted({1, 2, 3, d - 1, d}):
                    if slots < 1:
                        continue
                    ok = S.deadlock_free(pl, slots) if pl else True
                    if order == "paper" and slots < d - 1:
                        ok = False
                    if not ok:
                        with pytest.raises(sidp.SidpError):
                            sidp.Context(m, rank=r, world=d, slots=slots, order=order, alloc=False)
                        continue
                    c = sidp.Context(m, rank=r, world=d, slots=slots, order=order, alloc=False)
                    assert c.plan() == pl
                    assert [c.owner_of(l) for l in range(L)] == own
                    if pl:
                        assert c.schedule(3) == S.slot_schedule(pl, slots, 3)
                    c.destroy()


def test_stagger_ticks_match_oracle(sidp):
    for d in range(1, 9):
        m = MODELS["tiny"].with_layers(2 * d)
        for r in range(d):
            c = sidp.Context(m, rank=r, world=d, slots=2, alloc=False)
            assert c.stagger_ticks() == S.stagger_ticks(d, r)
            c.destroy()


def test_custom_owner_map_and_rejections(sidp):
    m = MODELS["tiny"]
    c = sidp.Context(m, rank=0, world=2, layer_owner=[1, 1, 0, 0], alloc=False)
    assert [c.owner_of(l) for l in range(4)] == [1, 1, 0, 0]
    assert c.plan() == [0, 1]
    c.destroy()
    bad = [dict(layer_owner=[0, 1, 2, 0]), dict(slots=0), dict(rank=2), dict(max_batch=0),
           dict(slot_parts=3),                              # granularity: 0, 1 or 2
           dict(slot_parts=2, fetch_engine="ce"),           # tiles live in the SM fetch's device ring
           dict(slot_parts=2, slots=5),                     # 5 slots x 4 parts > 16 ring entries
           dict(fetch_ce_share=1.0), dict(fetch_ce_share=-0.1),   # copy-engine share in [0, 1)
           dict(fetch_ce_share=0.3, slot_parts=2)]          # the hybrid fetch needs whole layers
    for kw in bad:
        kw = {"rank": 0, "world": 2, **kw}
        with pytest.raises(sidp.SidpError) as e:
            sidp.Context(m, alloc=False, **kw)
        assert e.value.status == -1     # SIDP_EINVAL
    for kw in (dict(slot_parts=2, slots=4), dict(slot_parts=2, slots=8, pool="ffn")):
        sidp.Context(m, rank=0, world=2, alloc=False, **kw).destroy()   # 16 ring entries: fine
    with pytest.raises(sidp.SidpError):  # PAPER order with S < d-1 deadlocks (C-S4)
        sidp.Context(m.with_layers(8), rank=1, world=4, slots=2, order="paper", alloc=False)


def test_host_calls_need_alloc(sidp):
    c = _ctx(sidp)
    import ctypes
    kv = sidp._abi.KV(None, None, None, 0)
    st = sidp._abi.lib().sidp_decode_layer(c.h, None, 1, 0, 0, ctypes.byref(kv), None)
    assert st == sidp._abi.SIDP_ESTATE
    c.destroy()


@pytest.mark.parametrize("h,I,C,max_seg,MT", [(5120, 25600, 74, 8, 1), (8192, 28672, 74, 6, 1),
                                              (256, 768, 74, 8, 1), (5120, 25600, 10, 3, 1),
                                              (5120, 25600, 74, 8, 2), (256, 768, 74, 8, 2)])
def test_fused_mlp_schedule_invariants(sidp, h, I, C, max_seg, MT):
    """Host list schedule of the fused gate/up -> down launch (no GPU), MT token tiles: every
    gate/up (tile, token tile) runs once, whole; each down (tile, token tile)'s k-range is
    partitioned exactly by its units, whose segment indices are 0..nseg-1; per pair all gate/up
    units precede its down units; and the makespan under the scheduler's own cost model
    (k-steps; down k-step k of token tile mt after gate/up tile (k, mt)) stays within 10% of the
    work lower bound (or the dependency bound) for the full-size shapes."""
    import ctypes
    G, nks1, D, nks2 = I // 128, h // 128, (h + 255) // 256, I // 128
    cap = G * MT + D * MT * max_seg + 8
    units = (ctypes.c_int32 * (4 * cap))()
    off = (ctypes.c_int32 * (C + 1))()
    nseg = (ctypes.c_int32 * (D * MT))()
    n = ctypes.c_int32()
    sidp._abi.check(sidp._abi.lib().sidp_test_mlp_schedule(G, nks1, D, nks2, C, max_seg, MT, units,
                                                          cap, off, nseg, ctypes.byref(n)), "schedule")
    U = [tuple(units[4 * i:4 * i + 4]) for i in range(n.value)]
    ph = lambda u: u[0] & 0xff
    seg = lambda u: (u[0] >> 8) & 0xff
    mt_ = lambda u: (u[0] >> 16) & 0xffff
    gate = sorted((u[1], mt_(u)) for u in U if ph(u) == 0)
    assert gate == sorted((g, m) for g in range(G) for m in range(MT))
    assert all(u[2:] == (0, nks1) for u in U if ph(u) == 0)
    per_tile = {}
    for u in U:
        if ph(u) == 1:
            per_tile.setdefault((u[1], mt_(u)), []).append((u[2], u[3], seg(u)))
    assert sorted(per_tile) == sorted((t, m) for t in range(D) for m in range(MT))
    for (t, m), parts in per_tile.items():
        ks = sorted((a, b) for a, b, _ in parts)
        assert ks[0][0] == 0 and ks[-1][1] == nks2
        assert all(ks[i][1] == ks[i + 1][0] for i in range(len(ks) - 1))
        assert sorted(sg for _, _, sg in parts) == list(range(len(parts))) == list(range(nseg[t * MT + m]))
        assert nseg[t * MT + m] <= max_seg
    done, free = {}, []
    for c in range(C):
        lst = U[off[c]:off[c + 1]]
        phases = [ph(u) for u in lst]
        assert phases == sorted(phases)
        t = 0.0
        for u in lst:
            if ph(u) == 0:
                t += nks1
                done[(u[1], mt_(u))] = t
        free.append(t)
    end = list(free)
    for c in range(C):
        t = free[c]
        for u in U[off[c]:off[c + 1]]:
            if ph(u) == 1:
                for k in range(u[2], u[3]):
                    t = max(t, done[(k, mt_(u))]) + 1
        end[c] = t
    work = MT * (G * nks1 + D * nks2)
    bound = max(work / C, max(done.values()) + 1)
    if C == 74 and h >= 5120:
        assert max(end) <= 1.10 * bound, (max(end), bound)


def test_paged_kv_binding_layout(sidp):
    """PagedKVCache (host side of sidp_kv.block_table): from_contiguous scatters each row's
    16-token blocks to a seeded permutation of the pool and to_contiguous gathers them back
    exactly; the ctypes struct carries the table, block size, row stride and pool size."""
    import torch
    m = MODELS["tiny"].with_layers(2)
    kv = sidp.KVCache(m, 3, 40, device="cpu")
    g = torch.Generator().manual_seed(3)
    kv.k.copy_(torch.randn(kv.k.shape, generator=g).to(torch.bfloat16))
    kv.v.copy_(torch.randn(kv.v.shape, generator=g).to(torch.bfloat16))
    kv.set_pos([5, 17, 33])
    pk = sidp.PagedKVCache.from_contiguous(kv, m, seed=9, spare=4)
    assert pk.max_blocks == 3 and pk.num_blocks == 3 * 3 + 4
    assert sorted(pk.table.flatten().tolist()) == sorted(set(pk.table.flatten().tolist()))
    for l in range(2):
        for which, ref in (("k", kv.k[l]), ("v", kv.v[l])):
            got = pk.to_contiguous(l, which)[:, :, :40]
            assert torch.equal(got, ref)
    c = pk.c()
    assert c.block_tokens == 16 and c.max_blocks == 3 and c.num_blocks == 13
    assert c.block_table == pk.table.data_ptr() and c.max_pos == 33
    assert kv.c().block_table is None


def test_prefill_rows():
    """Prefill's row layout (host logic of paper_2605_28095_b200.prefill): every prompt token is a
    row at position pos0[b] + i of its sequence; the last row of each sequence gives its next
    token."""
    import numpy as np
    from paper_2605_28095_b200.api import prefill_rows
    seq, pos, toks, last = prefill_rows(np.array([10, 0, 20]), [[1, 2], [3], [4, 5, 6]])
    assert seq.tolist() == [0, 0, 1, 2, 2, 2]
    assert pos.tolist() == [10, 11, 0, 20, 21, 22]
    assert toks.tolist() == [1, 2, 3, 4, 5, 6]
    assert last.tolist() == [1, 2, 5]
