"""Diag-only: write a copy of attention.cu with clock64 trace hooks in the backward kernel (CTA 0)
and an exported maestro_diag_trace(); build it with nvcc into _lib/diag/lib_<V>.so and read it
with scripts/attn_btrace.py.   python scripts/diag/make_btrace.py OUT.cu"""
import sys
from pathlib import Path

src = (Path(__file__).resolve().parents[2] / "paper_2605_10501_b200/csrc/attention.cu").read_text()
HDR = ('#include "tma_host.cuh"\n__device__ long long g_trace[20][1024];\n'
       '#define TR(k, idx) do { if (blockIdx.x == 0 && (idx) < 1024) g_trace[k][idx] = clock64(); } while (0)\n'
       'extern "C" int maestro_diag_trace(void* out) { return (int)cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)); }\n')
PATCHES = [
    ('#include "tma_host.cuh"\n', HDR),
    ('        if (nxt.valid) issue_s(nxt, gi + 1);\n        // dV += P^T dO\n        mbar_wait(p_ready, gi & 1);',
     '        if (nxt.valid) issue_s(nxt, gi + 1);\n        TR(2, gi);\n        // dV += P^T dO\n        mbar_wait(p_ready, gi & 1);\n        TR(0, gi);'),
    ('        umma_commit(p_free);\n', '        umma_commit(p_free);\n        TR(1, gi);\n'),
    ('        mbar_wait(ds_ready, gi & 1);\n        mbar_wait(dq_empty, (gi & 1) ^ 1);',
     '        mbar_wait(ds_ready, gi & 1);\n        TR(3, gi);\n        mbar_wait(dq_empty, (gi & 1) ^ 1);\n        TR(4, gi);'),
    ('        umma_commit(ds_free);\n', '        umma_commit(ds_free);\n        TR(5, gi);\n'),
    ('        if (nxt.valid) issue_dp(nxt, gi + 1);\n        cur = nxt;', '        if (nxt.valid) issue_dp(nxt, gi + 1);\n        TR(6, gi);\n        cur = nxt;'),
    ('        mbar_wait(s_full, gi & 1);\n        tc_fence_after();\n        uint32_t sr2[2][32];',
     '        mbar_wait(s_full, gi & 1);\n        if (warp == 2 && lane == 0) TR(7, gi);\n        tc_fence_after();\n        uint32_t sr2[2][32];'),
    ('        if (gi >= 1) mbar_wait(p_free, (gi - 1) & 1);  // dV(gi-1) has read P^T\n',
     '        if (gi >= 1) mbar_wait(p_free, (gi - 1) & 1);  // dV(gi-1) has read P^T\n        if (warp == 2 && lane == 0) TR(8, gi);\n'),
    ('        mbar_arrive(p_ready);\n        // ---- P2: dP^T -> dS^T\n        mbar_wait(dp_full, gi & 1);',
     '        mbar_arrive(p_ready);\n        if (warp == 2 && lane == 0) TR(9, gi);\n        // ---- P2: dP^T -> dS^T\n        mbar_wait(dp_full, gi & 1);\n        if (warp == 2 && lane == 0) TR(10, gi);'),
    ('        if (gi >= 1) mbar_wait(ds_free, (gi - 1) & 1);  // dQ(gi-1) has read the dS^T smem operand\n',
     '        if (gi >= 1) mbar_wait(ds_free, (gi - 1) & 1);  // dQ(gi-1) has read the dS^T smem operand\n        if (warp == 2 && lane == 0) TR(11, gi);\n'),
    ('        mbar_arrive(ds_ready);\n      }', '        mbar_arrive(ds_ready);\n        if (warp == 2 && lane == 0) TR(12, gi);\n      }'),
    ('        mbar_wait(dq_full, gi & 1);\n        tc_fence_after();\n        uint32_t qa[32], qb[32];',
     '        mbar_wait(dq_full, gi & 1);\n        if (warp == 10 && lane == 0) TR(13, gi);\n        tc_fence_after();\n        uint32_t qa[32], qb[32];'),
    ('          staged = true;\n        }', '          staged = true;\n        }\n        if (warp == 10 && lane == 0) TR(14, gi);'),
    ('        if (gi >= 1) mbar_wait(s_empty, (gi - 1) & 1);  // S^T(gi-1) is in the softmax registers\n',
     '        TR(15, gi);\n        if (gi >= 1) mbar_wait(s_empty, (gi - 1) & 1);  // S^T(gi-1) is in the softmax registers\n        TR(16, gi);\n'),
    ('        umma_commit(s_full);\n', '        umma_commit(s_full);\n        TR(17, gi);\n'),
    ('      auto issue_s = [&](const BwdCursor<CAUSAL>& c, int gi) {\n',
     '      auto issue_s = [&](const BwdCursor<CAUSAL>& c, int gi) {\n        TR(18, gi);\n'),
    ('        for (int kk = 0; kk < BKV / 16; ++kk)  // reduction over the 128 keys\n',
     '        TR(19, gi);\n#pragma unroll\n        for (int kk = 0; kk < BKV / 16; ++kk)  // reduction over the 128 keys\n'),
]
for old, new in PATCHES:
    assert old in src, old
    src = src.replace(old, new, 1)
Path(sys.argv[1]).write_text(src)
