"""Developer check of the fused tensor-core probe: raw MMA dot products of
the first CTA tile vs a float64 reference of the same split rows, candidate
counts, and the kernel time.

    python tools/probe_tc_dbg.py [K] [nq] [ma]
"""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import oracle as orc
from paper_1704_07355_b200 import _native, datagen

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 300
ma = int(sys.argv[3]) if len(sys.argv) > 3 else 16
d = 128
lib = _native.load_library()
lib.qadc_b200_debug_probe_tc.restype = ctypes.c_int
lib.qadc_b200_debug_probe_tc.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.c_int] + \
    [ctypes.c_void_p] * 5
test_seeds = len(sys.argv) > 4  # the seeds of test_probe_many_query_tiles_vs_oracle
cen = datagen.mixture_numpy(datagen.SIFT_LIKE, K, seed=K + nq if test_seeds else 3, stream=1)
qs = datagen.mixture_numpy(datagen.SIFT_LIKE, nq, seed=K if test_seeds else 3, stream=4)
dev = torch.device("cuda")
C, Q = torch.from_numpy(cen).to(dev), torch.from_numpy(qs).to(dev)
cells = torch.zeros((nq, ma), dtype=torch.int64, device=dev)
S = torch.zeros((128, 256), dtype=torch.float32, device=dev)
counts = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
mu = torch.zeros(d, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream().cuda_stream
rc = lib.qadc_b200_debug_probe_tc(C.data_ptr(), K, d, Q.data_ptr(), nq, ma, cells.data_ptr(),
                                  S.data_ptr(), counts.data_ptr(), mu.data_ptr(), st)
torch.cuda.synchronize()
print("rc", rc)
# float64 reference of the split products
m = mu.cpu().numpy().astype(np.float64)
qc = qs[:128].astype(np.float64) - m
cc = cen[:256].astype(np.float64) - m
ref = qc @ cc.T
got = S.cpu().numpy().astype(np.float64)
nqr = min(128, nq)
err = np.abs(got[:nqr] - ref[:nqr])
print("S[0,:4]", got[0, :4], "ref", ref[0, :4])
print("max abs err", err.max(), "rel to |q||c|", (err / (np.linalg.norm(qc[:nqr], axis=1)[:, None] *
                                                        np.linalg.norm(cc, axis=1)[None, :])).max())
# transposed / permuted checks
for name, cand in [("ref.T-ish", ref[:nqr, ::-1])]:
    print(name, np.abs(got[:nqr] - cand).max())
sl = int(counts[0].item())
nq_pad = (nq + 127) // 128 * 128
cn = counts[1:1 + sl * nq_pad].cpu().numpy().reshape(sl, nq_pad)[:, :nq]
print("slices", sl, "candidates per (slice, query): mean", cn.mean(), "max", cn.max())
got_c = cells.cpu().numpy()
nchk = nq if test_seeds else min(nq, 50)
badq = [i for i in range(nchk) if not np.array_equal(got_c[i], orc.probe(cen, qs[i], ma)[0])]
print(f"probe mismatches in {nchk} queries:", len(badq), badq[:10])
for i in badq[:3]:
    want = orc.probe(cen, qs[i], ma)[0]
    print("  q", i, "got", got_c[i][:8], "want", want[:8],
          "cands per slice", [int(cn[s_, i]) for s_ in range(sl)])
for _ in range(2):
    lib.qadc_b200_debug_probe_tc(C.data_ptr(), K, d, Q.data_ptr(), nq, ma, cells.data_ptr(),
                                 S.data_ptr(), counts.data_ptr(), mu.data_ptr(), st)
torch.cuda.synchronize()
t0 = time.perf_counter()
lib.qadc_b200_debug_probe_tc(C.data_ptr(), K, d, Q.data_ptr(), nq, ma, cells.data_ptr(),
                             S.data_ptr(), None, mu.data_ptr(), st)
torch.cuda.synchronize()
print("probe (incl. prepare) wall ms", (time.perf_counter() - t0) * 1e3)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    lib.qadc_b200_debug_probe_tc(C.data_ptr(), K, d, Q.data_ptr(), nq, ma, cells.data_ptr(),
                                 S.data_ptr(), None, mu.data_ptr(), st)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if e.device_time_total > 0:
        print(f"  {e.device_time_total / 1e3:9.3f} ms  x{e.count}  {e.key[:80]}")
