"""Time swmd_cost_build_batch_f32 alone at the c4 shape (V=100k, w=300, 64 queries
of 8-64 words): python scripts/gram_probe.py [reps]   (SWMD_LIB / SWMD_GRAM32 select the build / kernel)"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2107_06433_b200 import _lib  # noqa: E402
from paper_2107_06433_b200.device import device, stream_ptr  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(4)
V, dim = 100_000, 300
dev = device()
s = stream_ptr(dev)
E = torch.randn((V, dim), dtype=torch.float32, device=dev)
E /= E.norm(dim=1, keepdim=True)
norms = torch.empty(V, dtype=torch.float32, device=dev)
_lib.call("swmd_row_norms_f32", E.data_ptr(), V, dim, dim, norms.data_ptr(), s)
widths = rng.integers(8, 65, size=64)
words, col_word, off = [], [], 0
for w in widths:
    sel = np.sort(rng.choice(V, size=int(w), replace=False))
    blk = (int(w) + 7) // 8 * 8
    col_word += list(range(off, off + int(w))) + [-1] * (blk - int(w))
    words += list(sel)
    off += int(w)
LD = len(col_word)
words_d = torch.tensor(words, dtype=torch.int64, device=dev)
col_d = torch.tensor(col_word, dtype=torch.int32, device=dev)
K = torch.empty((V, LD), dtype=torch.float32, device=dev)
KM = torch.empty((V, LD), dtype=torch.float32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for r in range(reps + 2):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.call("swmd_cost_build_batch_f32", E.data_ptr(), V, dim, dim, words_d.data_ptr(),
              col_d.data_ptr(), LD, 10.0, norms.data_ptr(), None, 0, K.data_ptr(), KM.data_ptr(), s)
    b.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(a.elapsed_time(b))
print(f"LD {LD} gram {np.mean(ts):.3f} ms (min {np.min(ts):.3f}) lib {os.environ.get('SWMD_LIB', 'default')} "
      f"mode {os.environ.get('SWMD_GRAM32', 'tc5')}")
