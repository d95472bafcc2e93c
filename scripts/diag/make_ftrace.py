"""Diag-only: copy of attention.cu with clock64 trace hooks in the forward kernel (CTA 0, warp 2
lane 0 = softmax quadrant 2 half 0; warp 1 = MMA): per global KV tile g the s_full wait start/end
and the p_full arrive, per item the epilogue start/end.  python scripts/diag/make_ftrace.py OUT.cu"""
import sys
from pathlib import Path

src = (Path(__file__).resolve().parents[2] / "paper_2605_10501_b200/csrc/attention.cu").read_text()
HDR = ('#include "tma_host.cuh"\n__device__ long long g_trace[20][1024];\n'
       '#define TR(k, idx) do { if (blockIdx.x == 0 && (idx) < 1024) g_trace[k][idx] = clock64(); } while (0)\n'
       'extern "C" int maestro_diag_trace(void* out) { return (int)cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)); }\n')
W = "if (warp == 2 && lane == 0) "
PATCHES = [
    ('#include "tma_host.cuh"\n', HDR),
    ('      for (int i = 0; i < it.n_kv; ++i, ++g) {\n        const int b = g & 1;\n        mbar_wait(&s_full',
     f'      {W}TR(6, j);\n      if (warp == 2 && lane == 0 && blockIdx.x == 0 && j < 1024) g_trace[7][j] = it.n_kv;\n      for (int i = 0; i < it.n_kv; ++i, ++g) {{\n        const int b = g & 1;\n        mbar_wait(&s_full'),
    ('        mbar_wait(&s_full[b], (g >> 1) & 1);\n        tc_fence_after();\n        float s[64];',
     f'        {W}TR(0, g);\n        mbar_wait(&s_full[b], (g >> 1) & 1);\n        {W}TR(1, g);\n        tc_fence_after();\n        float s[64];'),
    ('        mbar_arrive(&p_full[b]);\n        if (i == 0 && pend) {\n          epilogue(pit, pj, pm, pl);\n          pend = false;\n        }',
     f'        mbar_arrive(&p_full[b]);\n        {W}TR(2, g);\n        if (i == 0 && pend) {{\n          {W}TR(3, j);\n          epilogue(pit, pj, pm, pl);\n          {W}TR(4, j);\n          pend = false;\n        }}\n        {W}TR(5, g);'),
]
for old, new in PATCHES:
    assert old in src, old
    src = src.replace(old, new, 1)
Path(sys.argv[1]).write_text(src)
