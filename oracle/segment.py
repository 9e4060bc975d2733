"""Reference implementation of the segmentation-guided initialisation reading
(Q24-Q26).  TEST INFRASTRUCTURE
ONLY: plain Python, obviously-correct loops, used to check the library's
host C++ (smoe_segment / smoe_segment_init) label for label.

The paper cites a "modified DBSCAN" region clustering with pixel difference
thresholds 10 and 20 without giving it; the steps below
are the reading DESIGN.md states, in its order:
  1. row-major seeds; breadth-first growth over 4-neighbours (right, down,
     left, up); a pixel joins when max_c |255 p_c - mean_c| <= threshold,
     the region mean (0-255 scale) updated as a running mean;
  2. regions smaller than min_size, lowest id first and repeated until none
     changes, merge into the adjacent region with the smallest max-channel
     mean difference (ties: lowest id), size-weighted means;
  3. ids relabelled 0..N-1 in row-major order of first appearance.
"""
from collections import deque

import numpy as np


def segment(image, threshold, min_size):
    img = 255.0 * np.asarray(image, np.float64)
    C, H, W = img.shape
    lab = -np.ones((H, W), np.int64)
    means, sizes = [], []
    nbrs = ((1, 0), (0, 1), (-1, 0), (0, -1))
    for sy in range(H):
        for sx in range(W):
            if lab[sy, sx] >= 0:
                continue
            rid = len(means)
            m = img[:, sy, sx].copy()
            n = 1
            lab[sy, sx] = rid
            q = deque([(sx, sy)])
            while q:
                x, y = q.popleft()
                for dx, dy in nbrs:
                    xx, yy = x + dx, y + dy
                    if not (0 <= xx < W and 0 <= yy < H) or lab[yy, xx] >= 0:
                        continue
                    if np.max(np.abs(img[:, yy, xx] - m)) <= threshold:
                        lab[yy, xx] = rid
                        n += 1
                        m = m + (img[:, yy, xx] - m) / n
                        q.append((xx, yy))
            means.append(m)
            sizes.append(n)
    R = len(means)
    parent = list(range(R))

    def find(r):
        while parent[r] != r:
            r = parent[r]
        return r

    adj = [set() for _ in range(R)]
    for y in range(H):
        for x in range(W):
            a = lab[y, x]
            for xx, yy in ((x + 1, y), (x, y + 1)):
                if xx < W and yy < H and lab[yy, xx] != a:
                    adj[a].add(int(lab[yy, xx]))
                    adj[int(lab[yy, xx])].add(int(a))
    changed = True
    while changed:
        changed = False
        for r in range(R):
            if find(r) != r or sizes[r] >= min_size:
                continue
            nb = sorted({find(o) for o in adj[r]} - {r})
            if not nb:
                continue
            diffs = [np.max(np.abs(means[o] - means[r])) for o in nb]
            best = nb[int(np.argmin(diffs))]
            n = sizes[r] + sizes[best]
            means[best] = (means[best] * sizes[best] + means[r] * sizes[r]) / n
            sizes[best] = n
            parent[r] = best
            adj[best] |= {o for o in nb if o != best}
            adj[r] = set()
            changed = True
    out = np.empty((H, W), np.int64)
    newid = {}
    for y in range(H):
        for x in range(W):
            r = find(int(lab[y, x]))
            if r not in newid:
                newid[r] = len(newid)
            out[y, x] = newid[r]
    return out, len(newid)


def allocate(labels, n_segments, K):
    """Kernels per segment: max(1, floor(K |R| / HW)) plus largest-remainder
    top-up to exactly K (ties: lowest id); trimmed from the largest segments
    (keeping >= 1) when the floors of 1 overshoot."""
    sizes = np.bincount(np.asarray(labels).ravel(), minlength=n_segments)
    if K < n_segments:
        raise ValueError("TooFewKernels")
    share = K * sizes / sizes.sum()
    cnt = np.maximum(1, np.floor(share)).astype(np.int64)
    rem = share - np.floor(share)
    order = sorted(range(n_segments), key=lambda s: -rem[s])
    i = 0
    while cnt.sum() < K:
        cnt[order[i % n_segments]] += 1
        i += 1
    order = sorted(range(n_segments), key=lambda s: -sizes[s])
    i = 0
    while cnt.sum() > K:
        s = order[i % n_segments]
        if cnt[s] > 1:
            cnt[s] -= 1
        i += 1
    return cnt
