"""Recall harness on the GPU: exact ground truth for
BASELINE-sized bases and the reference's recall definition.

Mirrors /root/reference/pkg/src/qadc/synth.py:45-70 (`ground_truth`: GEMM
preselect, then float64 re-measure, ties to the lower id) and
bench.py:110-122 (`recall_at`: fraction of queries whose true nearest
neighbour appears in the first R' results).
"""

from __future__ import annotations

import numpy as np


def ground_truth(base_chunks, queries, depth: int = 1, preselect: int = 64, device="cuda"):
    """Exact `depth` nearest base ids per query. `base_chunks` yields
    (offset, float32 CUDA tensor (n, d)) chunks of the base in id order.
    Candidates come from a float32 GEMM expansion (top `preselect` per
    chunk), then are re-measured exactly in float64."""
    import torch

    q = torch.as_tensor(np.ascontiguousarray(queries, np.float32), device=device)
    qn = (q.double() ** 2).sum(1)
    cand_d, cand_i = [], []
    for off, X in base_chunks:
        d2 = (X.double() ** 2).sum(1)[None, :].float() - 2.0 * (q @ X.T) + qn[:, None].float()
        k = min(preselect, X.shape[0])
        v, i = torch.topk(d2, k, dim=1, largest=False)
        exact = ((X[i].double() - q[:, None, :].double()) ** 2).sum(2)
        cand_d.append(exact)
        cand_i.append(i + off)
    d = torch.cat(cand_d, 1)
    i = torch.cat(cand_i, 1)
    # ties to the lower id: sort by id, then stably by distance
    o = torch.argsort(i, dim=1, stable=True)
    d, i = torch.gather(d, 1, o), torch.gather(i, 1, o)
    o = torch.argsort(d, dim=1, stable=True)
    return torch.gather(i, 1, o)[:, :depth].cpu().numpy()


def recall_at(result_ids: np.ndarray, gt_first: np.ndarray, r: int) -> float:
    """bench.py:110-122: fraction of queries whose true 1-NN is in the
    first r result ids."""
    hits = [gt_first[i] in result_ids[i, :r] for i in range(result_ids.shape[0])]
    return float(np.mean(hits)) if hits else 0.0
