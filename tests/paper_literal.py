"""The paper's own tensor programs, restated literally in torch (TEST-ONLY).

These are independent routes to the oracle's results: they follow the paper's
algorithms step by step in its order and notation, so a test that finds
oracle == paper_literal on random small inputs pins the oracle's plain
definition to what the paper computes. Variant switches reproduce the paper's
conflicting texts so the tests can show which
reading is the correct one.

  alg1_sort_based_join   PAPER.md:286-338 (Alg. 1), long form PAPER.md:102-165
  pkfk_join_macro        PAPER.md:55-100 (PK-FK join macro)
  alg2_aggregation       PAPER.md:340-367 (Alg. 2), long form PAPER.md:247-284
  filter_bm / filter_sv  PAPER.md:832-834 (Listing 1), PAPER.md:846-849 (Listing 2)
"""

import math

import numpy as np
import torch


def alg1_sort_based_join(left, right, descending=False, bucketize_right=True, remainder_by="right",
                         trace=None):
    """Alg. 1 line by line. Keys must be non-negative integers (bincount domain)."""
    left = torch.as_tensor(np.asarray(left, dtype=np.int64))
    right = torch.as_tensor(np.asarray(right, dtype=np.int64))
    # l.2-3: sort join keys (reading R1: stable)
    left_s, leftIdx = torch.sort(left, descending=descending, stable=True)
    right_s, rightIdx = torch.sort(right, descending=descending, stable=True)
    # l.4: histograms (both over a common domain so that mul is defined, reading R5)
    K = int(max(left.max().item() if left.numel() else 0, right.max().item() if right.numel() else 0)) + 1
    leftHist = torch.bincount(left_s, minlength=K)
    rightHist = torch.bincount(right_s, minlength=K)
    # l.5
    histMul = leftHist * rightHist
    # l.6-8
    cumLeftHist = torch.cumsum(leftHist, dim=0)
    cumRightHist = torch.cumsum(rightHist, dim=0)
    cumHistMul = torch.cumsum(histMul, dim=0)
    # l.9-10
    outSize = int(cumHistMul[-1].item())
    offset = torch.arange(outSize)
    # l.11 (reading R3: right=True as in the long form)
    outBucket = torch.bucketize(offset, cumHistMul, right=bucketize_right)
    # l.12
    offset = offset - (cumHistMul[outBucket] - histMul[outBucket])
    # l.13-14 (reading R4: div and remainder by rightHist)
    div = torch.div(offset, rightHist[outBucket], rounding_mode="floor")
    rem_div = rightHist if remainder_by == "right" else leftHist
    rem = torch.remainder(offset, rem_div[outBucket])
    leftOutIdx = leftIdx[cumLeftHist[outBucket] - leftHist[outBucket] + div]
    rightOutIdx = rightIdx[cumRightHist[outBucket] - rightHist[outBucket] + rem]
    if trace is not None:
        trace.update(leftHist=leftHist.tolist(), rightHist=rightHist.tolist(), histMul=histMul.tolist(),
                     cumHistMul=cumHistMul.tolist(), outSize=outSize, outBucket=outBucket.tolist())
    return leftOutIdx.numpy(), rightOutIdx.numpy()


def pkfk_join_macro(left, right, pad="safe"):
    """PK-FK macro literally; returns (leftOutputIndex, rightOutputIndex).

    pad="literal" uses minVal-1 with minVal = min(left), which can
    index out of range (reading R8); pad="safe" uses min(left U right) - 1.
    """
    left = torch.as_tensor(np.asarray(left, dtype=np.int64))
    right = torch.as_tensor(np.asarray(right, dtype=np.int64))
    left_s, leftIndex = torch.sort(left, descending=True, stable=True)
    right_s, rightIndex = torch.sort(right, descending=True, stable=True)
    n = left_s.shape[0]
    nPrime = 1
    while nPrime <= n:          # smallestPowerOfTwoGreaterThan(n)
        nPrime *= 2
    if pad == "literal":
        minVal = int(left.min().item())
    else:
        minVal = int(torch.cat([left, right]).min().item())
    paddedLeft = torch.cat([left_s, torch.full((nPrime - n,), minVal - 1, dtype=torch.int64)])
    offset = nPrime // 2
    bins = right_s <= paddedLeft[offset]
    pos = bins.long() * offset
    offset = (offset + 1) // 2
    for _ in range(int(math.log2(nPrime))):
        bins = right_s <= torch.index_select(paddedLeft, 0, pos + offset)
        pos = pos + bins.long() * offset
        offset = offset // 2
    mask = right_s == torch.index_select(left_s, 0, pos)   # PAPER.md:81 indexes `left`
    pos = torch.masked_select(pos, mask)
    leftOutputIndex = torch.index_select(leftIndex, 0, pos)
    rightOutputIndex = torch.masked_select(rightIndex, mask)
    return leftOutputIndex.numpy(), rightOutputIndex.numpy()


def alg2_aggregation(key_cols, value_cols):
    """Alg. 2: cat -> row sort (reading R12: lexicographic,
    column 0 most significant) -> permute -> uniqueConsecutive(inverse) ->
    evaluate (sum per value column via scatter_add, count via bincount).
    Returns (unique key rows [G x m], sums [n_values x G] python ints, counts)."""
    grps = torch.stack([torch.as_tensor(np.asarray(c, dtype=np.int64)) for c in key_cols], dim=1)
    # l.3: lexicographic row sort, stable: np.lexsort sorts by the LAST key first
    perm = np.lexsort(tuple(grps[:, j].numpy() for j in reversed(range(grps.shape[1]))))
    perm = torch.as_tensor(perm)
    grps = grps[perm]
    data = [torch.as_tensor(np.asarray(c, dtype=np.int64))[perm] for c in value_cols]   # l.4
    uniq, inv = torch.unique_consecutive(grps, dim=0, return_inverse=True)             # l.5
    G = uniq.shape[0]
    sums = []
    for col in data:
        # exact sums: accumulate as python ints per group (scatter in object space)
        acc = [0] * G
        for g, v in zip(inv.tolist(), col.tolist()):
            acc[g] += v
        sums.append(acc)
    counts = torch.bincount(inv, minlength=G).tolist()
    return uniq.numpy(), sums, counts


def filter_bm(col, op, c):
    """Listing 1: mask = torch.<op>(col, c); output = masked_select(col, mask)."""
    t = torch.as_tensor(np.asarray(col))
    mask = getattr(torch, op)(t, c)
    return mask, torch.masked_select(t, mask)


def filter_sv(col, op, c):
    """Listing 2 with reading R20 (index_select by idx, not mask)."""
    t = torch.as_tensor(np.asarray(col))
    mask = getattr(torch, op)(t, c)
    idx = torch.nonzero(mask).flatten()
    return idx, torch.index_select(t, 0, idx)
