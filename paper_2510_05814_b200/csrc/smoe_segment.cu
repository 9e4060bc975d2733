// smoe_segment.cu -- segmentation-guided kernel initialisation (host C++).
//
// SURVEY §8(f) f4.  The paper initialises denoising fits from segments found
// by "modified DBSCAN ... a region-based clustering method ... from pixel RGB
// similarity" with "pixel difference thresholds of 10 and 20" (P:264-277,
// P:424) and distributes the kernel budget so that each kernel's block set
// grows with its segment, |B_j| ~ |R_j| / n_k (Eq. 9).  The cited algorithm
// is not given, so this follows the reading written down in SPEC S:417-438
// (Q24-Q26):
//   * 4-connected region growing from row-major seeds; a pixel joins when the
//     max-channel absolute difference to the region's running mean, on the
//     0-255 scale, is <= threshold; BFS in FIFO order, neighbours visited
//     right, down, left, up;
//   * regions smaller than min_size merge into the 4-adjacent region with the
//     closest mean (max-channel difference; ties: lowest id), smallest-id
//     first, until none remains;
//   * kernels per segment: max(1, floor(L |R|/N_px)) plus largest-remainder
//     top-up to exactly L (ties: lowest id); centres uniform over the
//     segment's pixels (+-0.5 px jitter), isotropic scale, expert = segment
//     mean colour, log_pi = 0, slopes 0.
// Host code: runs once before a fit; not on the per-iteration hot path.
#include "smoe.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <set>
#include <vector>

namespace {

struct SplitMix {
    uint64_t s;
    uint64_t next()
    {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }   // [0,1)
};

}  // namespace

extern "C" {

smoe_status smoe_segment(const float *image, int H, int W, int C, float threshold, int min_size, int *labels,
                         int *n_segments)
{
    if (!image || !labels || !n_segments || H < 1 || W < 1 || C < 1 || !(threshold > 0.f) || min_size < 1)
        return SMOE_ERR_INVALID_ARG;
    const size_t npx = (size_t)H * W;
    std::vector<int> lab(npx, -1);
    std::vector<std::vector<double>> mean;   // per region, 0-255 scale
    std::vector<long long> size;
    auto pix = [&](size_t i, int c) { return 255.0 * (double)image[(size_t)c * npx + i]; };
    const int dx4[4] = {1, 0, -1, 0}, dy4[4] = {0, 1, 0, -1};
    std::deque<size_t> q;
    for (size_t s = 0; s < npx; s++) {
        if (lab[s] >= 0) continue;
        int id = (int)mean.size();
        std::vector<double> m(C);
        for (int c = 0; c < C; c++) m[c] = pix(s, c);
        long long n = 1;
        lab[s] = id;
        q.clear();
        q.push_back(s);
        while (!q.empty()) {
            size_t i = q.front();
            q.pop_front();
            int x = (int)(i % W), y = (int)(i / W);
            for (int d = 0; d < 4; d++) {
                int xx = x + dx4[d], yy = y + dy4[d];
                if (xx < 0 || yy < 0 || xx >= W || yy >= H) continue;
                size_t j = (size_t)yy * W + xx;
                if (lab[j] >= 0) continue;
                double diff = 0.0;
                for (int c = 0; c < C; c++) diff = std::max(diff, std::fabs(pix(j, c) - m[c]));
                if (diff <= threshold) {
                    lab[j] = id;
                    n++;
                    for (int c = 0; c < C; c++) m[c] += (pix(j, c) - m[c]) / (double)n;
                    q.push_back(j);
                }
            }
        }
        mean.push_back(m);
        size.push_back(n);
    }
    // merge small regions into their closest 4-adjacent neighbour: region
    // adjacency sets (merged small-into-large) + union-find over region ids
    int R = (int)mean.size();
    std::vector<int> parent(R);
    for (int r = 0; r < R; r++) parent[r] = r;
    auto find = [&](int r) {
        while (parent[r] != r) r = parent[r] = parent[parent[r]];
        return r;
    };
    std::vector<std::set<int>> adj(R);
    for (size_t i = 0; i < npx; i++) {
        int x = (int)(i % W), y = (int)(i / W);
        if (x + 1 < W && lab[i + 1] != lab[i]) { adj[lab[i]].insert(lab[i + 1]); adj[lab[i + 1]].insert(lab[i]); }
        if (y + 1 < H && lab[i + W] != lab[i]) { adj[lab[i]].insert(lab[i + W]); adj[lab[i + W]].insert(lab[i]); }
    }
    for (bool changed = true; changed;) {
        changed = false;
        for (int r = 0; r < R; r++) {
            if (find(r) != r || size[r] >= min_size) continue;
            int best = -1;
            double bd = 1e300;
            std::set<int> nb;
            for (int o : adj[r]) {
                int oo = find(o);
                if (oo != r) nb.insert(oo);
            }
            for (int o : nb) {
                double diff = 0.0;
                for (int c = 0; c < C; c++) diff = std::max(diff, std::fabs(mean[o][c] - mean[r][c]));
                if (diff < bd) { bd = diff; best = o; }   // nb ascending: ties keep the lowest id
            }
            if (best < 0) continue;   // the only region left
            long long n = size[r] + size[best];
            for (int c = 0; c < C; c++) mean[best][c] = (mean[best][c] * size[best] + mean[r][c] * size[r]) / n;
            size[best] = n;
            parent[r] = best;
            if (adj[best].size() < nb.size()) std::swap(adj[best], nb);
            for (int o : nb) if (o != best) adj[best].insert(o);
            std::set<int>().swap(adj[r]);
            changed = true;
        }
    }
    std::vector<int> newid(R, -1);
    int N = 0;
    for (size_t i = 0; i < npx; i++) {
        int r = find(lab[i]);
        if (newid[r] < 0) newid[r] = N++;
        labels[i] = newid[r];
    }
    *n_segments = N;
    return SMOE_OK;
}

smoe_status smoe_segment_init(const float *image, int H, int W, int C, const int *labels, int n_segments, int K,
                              int expert_order, unsigned long long seed, float scale_px, float *mu, float *chol,
                              float *log_pi, float *expert)
{
    if (!image || !labels || !mu || !chol || !log_pi || !expert || n_segments < 1 || K < 1 ||
        !(expert_order == 0 || expert_order == 1) || !(scale_px > 0.f) || H < 1 || W < 1 || C < 1)
        return SMOE_ERR_INVALID_ARG;
    if (K < n_segments) return SMOE_ERR_INVALID_ARG;   // SPEC TooFewKernels
    const size_t npx = (size_t)H * W;
    std::vector<std::vector<size_t>> members(n_segments);
    for (size_t i = 0; i < npx; i++) {
        int l = labels[i];
        if (l < 0 || l >= n_segments) return SMOE_ERR_INVALID_ARG;
        members[l].push_back(i);
    }
    // every segment id must own a pixel (its kernels are placed on its pixels
    // and its expert is its mean colour)
    for (int s = 0; s < n_segments; s++)
        if (members[s].empty()) return SMOE_ERR_INVALID_ARG;
    // budget: max(1, floor(K |R|/N)) then largest remainder to exactly K
    std::vector<long long> cnt(n_segments);
    std::vector<double> rem(n_segments);
    long long tot = 0;
    for (int s = 0; s < n_segments; s++) {
        double share = (double)K * (double)members[s].size() / (double)npx;
        cnt[s] = std::max(1LL, (long long)std::floor(share));
        rem[s] = share - std::floor(share);
        tot += cnt[s];
    }
    std::vector<int> order(n_segments);
    for (int s = 0; s < n_segments; s++) order[s] = s;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rem[a] > rem[b]; });
    for (int i = 0; tot < K; i = (i + 1) % n_segments) { cnt[order[i]]++; tot++; }
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return members[a].size() > members[b].size(); });
    for (int i = 0; tot > K; i = (i + 1) % n_segments)
        if (cnt[order[i]] > 1) { cnt[order[i]]--; tot--; }
    // kernels
    SplitMix rng{seed};
    const int E = 1 + 2 * expert_order;
    int k = 0;
    for (int s = 0; s < n_segments; s++) {
        std::vector<double> m(C, 0.0);
        for (size_t i : members[s])
            for (int c = 0; c < C; c++) m[c] += image[(size_t)c * npx + i];
        for (int c = 0; c < C; c++) m[c] /= (double)members[s].size();
        for (long long t = 0; t < cnt[s]; t++, k++) {
            size_t i = members[s][(size_t)(rng.uniform() * members[s].size())];
            mu[2 * k] = (float)((double)(i % W) + rng.uniform() - 0.5);
            mu[2 * k + 1] = (float)((double)(i / W) + rng.uniform() - 0.5);
            chol[3 * k] = scale_px; chol[3 * k + 1] = 0.f; chol[3 * k + 2] = scale_px;
            log_pi[k] = 0.f;
            for (int c = 0; c < C; c++) {
                expert[((size_t)k * C + c) * E] = (float)m[c];
                for (int e = 1; e < E; e++) expert[((size_t)k * C + c) * E + e] = 0.f;
            }
        }
    }
    return SMOE_OK;
}

}  // extern "C"
