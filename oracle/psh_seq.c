/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's sequential PSH claim loop, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER. Nothing on the product path links or calls this file.
 *
 * Follows:
 *   bucketswin/_kernels.py:17-24   _morton      (x at bit 3k, y at 3k+1, z at 3k+2)
 *   bucketswin/_kernels.py:27-38   _hash        (xor / morton, //S_div, strict -1, %K)
 *   bucketswin/_kernels.py:41-66   _probe_claim (clamp to [0,vmax], claim if count<S)
 *   bucketswin/_kernels.py:69-90   assign_one_stage (direct, probe, recycle K)
 *   bucketswin/bucketing.py:294-305 per-batch private K+1 counters, batch-major
 *
 * Batches never share counters, so walking points in global index order with
 * ctr = counts + batch[i]*(K+1) is the same computation as the reference's
 * batch-by-batch loop over np.flatnonzero(batch == b).
 */
#include <stdint.h>

static int64_t morton3(int64_t x, int64_t y, int64_t z, int bits) {
    int64_t code = 0;
    for (int k = 0; k < bits; ++k) {
        code |= ((x >> k) & 1) << (3 * k);
        code |= ((y >> k) & 1) << (3 * k + 1);
        code |= ((z >> k) & 1) << (3 * k + 2);
    }
    return code;
}

/* kind: 0 xor-mod, 1 xor-div, 2 zorder-mod, 3 zorder-div (hashing.py:19) */
int64_t oracle_hash1(int64_t x, int64_t y, int64_t z, int kind, int64_t K,
                     int64_t S_div, int bits, int strict) {
    int64_t key = (kind <= 1) ? (x ^ y ^ z) : morton3(x, y, z, bits);
    if (kind == 1 || kind == 3) {
        key = key / S_div;               /* key >= 0: C '/' == numpy '//' */
        if (strict && key >= K) return -1;
    }
    return key % K;
}

static inline int64_t clampv(int64_t v, int64_t hi) {
    return v < 0 ? 0 : (v > hi ? hi : v);
}

/*
 * vox:     (n,3) int64, non-negative, < 2^bits
 * home:    (n)   int64 home bucket (hash of vox)
 * batch:   (n)   int64 batch id or NULL
 * offsets: (P,3) int64 probe offsets
 * outputs: bucket_id (n), bucket_offset (n), counts (nbatch*(K+1)) zeroed here
 */
void oracle_psh_assign(const int64_t *vox, const int64_t *home, const int64_t *batch,
                       int64_t n, int64_t nbatch, int64_t K, int64_t S, int kind,
                       int64_t S_div, int bits, int strict, const int64_t *offsets,
                       int64_t P, int64_t max_probes, int64_t *bucket_id,
                       int64_t *bucket_offset, int64_t *counts) {
    const int64_t W = K + 1;
    const int64_t vmax = ((int64_t)1 << bits) - 1;
    const int64_t np_ = max_probes < P ? max_probes : P;
    for (int64_t s = 0; s < nbatch * W; ++s) counts[s] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t *ctr = counts + (batch ? batch[i] : 0) * W;
        int64_t h = home[i];
        if (ctr[h] < S) {
            bucket_id[i] = h;
            bucket_offset[i] = ctr[h]++;
            continue;
        }
        int64_t got = -1;
        for (int64_t p = 0; p < np_ && got < 0; ++p) {
            int64_t x = clampv(vox[3 * i + 0] + offsets[3 * p + 0], vmax);
            int64_t y = clampv(vox[3 * i + 1] + offsets[3 * p + 1], vmax);
            int64_t z = clampv(vox[3 * i + 2] + offsets[3 * p + 2], vmax);
            int64_t c = oracle_hash1(x, y, z, kind, K, S_div, bits, strict);
            if (c >= 0 && ctr[c] < S) got = c;
        }
        if (got < 0) got = K;            /* recycle: unbounded */
        bucket_id[i] = got;
        bucket_offset[i] = ctr[got]++;
    }
}
