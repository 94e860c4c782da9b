// Device-side planning: attention scope tables for one bucket-swin round and
// pooling tile tables, built from the PSH counts/bases already in HBM (no
// host round trip of per-scope data).
//
// Scope construction follows bw/attention.py:84-117 (build_schedule) over the
// split bucket table of bw/bucketing.py:147-166: table entry e < K is bucket e
// (start base[e], length counts[e]); entry K + j is recycle chunk j (start
// base[K] + j*S, length min(S, r - j*S)).  Round t rotates by off = (t*shift)
// mod W; scope (chunk, lane) holds positions chunk*W*stride + lane + j*stride
// (< min(nb, (chunk+1)*W*stride)).  Adjacent non-empty buckets are merged into
// one physical segment (bw/attention.py:120-139 ranges, concatenated).
#include "f3d_common.cuh"

namespace f3d {
namespace plan {

constexpr int kThreads = 1024;

// block-wide exclusive scan of one int per thread; returns the total
__device__ int block_excl_scan(int v, int& total, int* sh /* >= 33 ints */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int incl = warp_incl_scan(v);
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        int x = lane < nw ? sh[lane] : 0;
        const int xi = warp_incl_scan(x);
        sh[lane] = xi - x;
        if (lane == 31) sh[32] = xi;
    }
    __syncthreads();
    const int res = sh[w] + incl - v;
    total = sh[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kThreads) plan_round_kernel(
    const int32_t* __restrict__ counts, const int32_t* __restrict__ base, int K, int S, int nb_cap,
    int W, int stride, int off0, int off_step, int64_t round_stride, int nscopes,
    int32_t* scope_seg, int32_t* scope_nseg, int32_t* seg_start, int32_t* seg_vstart,
    int32_t* scope_len, int32_t* scope_order, int32_t* work, int max_work, int qstep,
    int32_t* live) {
    pdl_wait();
    // block t plans round t: rotation off0 + t*off_step, outputs round_stride apart
    const int off = (off0 + (int)blockIdx.x * off_step) % W;
    {
        const int64_t o = (int64_t)blockIdx.x * round_stride;
        scope_seg += o;
        scope_nseg += o;
        seg_start += o;
        seg_vstart += o;
        scope_len += o;
        scope_order += o;
        work += o;
        live += o;
    }
    __shared__ int sh[40];
    __shared__ int s_maxlen;
    const int span = W * stride;
    const int r = counts[K];
    const int rb = base[K];
    // table size from the device counts: K buckets + ceil(r/S) recycle chunks
    // (bw/bucketing.py:147-166); nb_cap (host bound) sized the scope arrays
    const int nb = K + (r + S - 1) / S;
    if (threadIdx.x == 0) s_maxlen = 0;
    __syncthreads();
    int carry_live = 0, carry_work = 0;
    for (int s0 = 0; s0 < nscopes; s0 += kThreads) {
        const int s = s0 + threadIdx.x;
        int v = 0;
        if (s < nscopes) {
            const int chunk = s / stride, lane = s - chunk * stride;
            const int pend = min(nb, (chunk + 1) * span);
            int nseg = 0, last_end = -1;
            for (int j = 0; j < W; ++j) {
                const int p = chunk * span + lane + j * stride;
                if (p >= pend) break;
                const int b = (p + off) % nb;
                int st, ln;
                if (b < K) {
                    st = base[b];
                    ln = counts[b];
                } else {
                    const int jj = b - K;
                    st = rb + jj * S;
                    ln = min(S, r - jj * S);
                }
                if (ln <= 0) continue;
                if (nseg > 0 && st == last_end) {
                    // adjacent bucket: extend the current segment
                } else {
                    seg_start[s * W + nseg] = st;
                    seg_vstart[s * W + nseg] = v;
                    ++nseg;
                }
                last_end = st + ln;
                v += ln;
            }
            scope_seg[s] = s * W;
            scope_nseg[s] = nseg;
            scope_len[s] = v;
            atomicMax(&s_maxlen, v);
        }
        int tot_live, tot_work;
        const int is_live = v > 0 ? 1 : 0;
        const int nt = v / qstep;                    // full query groups first
        const int pl = block_excl_scan(is_live, tot_live, sh) + carry_live;
        const int pw = block_excl_scan(nt, tot_work, sh) + carry_work;
        if (is_live) scope_order[pl] = s;
        for (int q = 0; q < nt; ++q)
            if (pw + q < max_work) {
                work[2 * (pw + q)] = s;
                work[2 * (pw + q) + 1] = q * qstep;
            }
        carry_live += tot_live;
        carry_work += tot_work;
    }
    // then every scope's partial last group (fewer query rows): with the
    // attention kernels' dynamic item counter the smaller items come last
    for (int s0 = 0; s0 < nscopes; s0 += kThreads) {
        const int s = s0 + threadIdx.x;
        const int v = s < nscopes ? scope_len[s] : 0;   // written by this thread above
        const int part = (v % qstep) ? 1 : 0;
        int tot_part;
        const int pw = block_excl_scan(part, tot_part, sh) + carry_work;
        if (part && pw < max_work) {
            work[2 * pw] = s;
            work[2 * pw + 1] = (v / qstep) * qstep;
        }
        carry_work += tot_part;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        live[0] = min(carry_work, max_work);
        live[1] = carry_live;
        live[2] = s_maxlen;
        // 1: window_w exceeds num_buckets (bw/attention.py:104); 2: table
        // larger than the capacity the host planned for; 4: work list cut
        live[3] = (W > nb ? 1 : 0) | (nb > nb_cap ? 2 : 0) | (carry_work > max_work ? 4 : 0);
        live[4] = 0;      // attention scheduler: next item, CTAs done (reset by the kernel)
        live[5] = 0;
    }
}

// Pool tiles: slot c's rows split into ceil(count/cap) tiles of <= cap rows
// in scatter order (bw/pooling.py:211-225); out = first pooled row.
__global__ void __launch_bounds__(kThreads) plan_pool_kernel(
    const int32_t* __restrict__ counts, const int32_t* __restrict__ base, int nslots, int cap,
    int rho, int32_t* tile_start, int32_t* tile_m, int32_t* tile_out, int32_t* totals) {
    __shared__ int sh[40];
    int carry_t = 0, carry_o = 0;
    for (int c0 = 0; c0 < nslots; c0 += kThreads) {
        const int c = c0 + threadIdx.x;
        const int cnt = c < nslots ? counts[c] : 0;
        const int nt = (cnt + cap - 1) / cap;
        const int full = cnt / cap, rem = cnt - full * cap;
        const int pooled = full * ((cap + rho - 1) / rho) + (rem + rho - 1) / rho;
        int tt, to;
        const int pt = block_excl_scan(nt, tt, sh) + carry_t;
        const int po = block_excl_scan(pooled, to, sh) + carry_o;
        if (c < nslots) {
            int o = po;
            for (int k = 0; k < nt; ++k) {
                const int m = min(cap, cnt - k * cap);
                tile_start[pt + k] = base[c] + k * cap;
                tile_m[pt + k] = m;
                tile_out[pt + k] = o;
                o += (m + rho - 1) / rho;
            }
        }
        carry_t += tt;
        carry_o += to;
    }
    if (threadIdx.x == 0) {
        totals[0] = carry_t;
        totals[1] = carry_o;
    }
}

}  // namespace plan
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_plan_round(const int32_t* counts, const int32_t* base, int K, int S, int nb_cap,
                              int W, int stride, int off, int nscopes, int32_t* scope_seg,
                              int32_t* scope_nseg, int32_t* seg_start, int32_t* seg_vstart,
                              int32_t* scope_len, int32_t* scope_order, int32_t* work,
                              int max_work, int qstep, int32_t* live, void* stream) {
    if (K < 1 || S < 1 || nb_cap < 1 || W < 1 || stride < 1 || off < 0 || nscopes < 1 ||
        max_work < 0 || qstep < 16)
        return F3D_ERR_CONFIG;
    plan::plan_round_kernel<<<1, plan::kThreads, 0, (cudaStream_t)stream>>>(
        counts, base, K, S, nb_cap, W, stride, off, 0, 0, nscopes, scope_seg, scope_nseg,
        seg_start, seg_vstart, scope_len, scope_order, work, max_work, qstep, live);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_plan_rounds(const int32_t* counts, const int32_t* base, int K, int S,
                               int nb_cap, int W, int stride, int shift, int nrounds,
                               int64_t round_stride, int nscopes, int32_t* scope_seg,
                               int32_t* scope_nseg, int32_t* seg_start, int32_t* seg_vstart,
                               int32_t* scope_len, int32_t* scope_order, int32_t* work,
                               int max_work, int qstep, int32_t* live, void* stream) {
    if (K < 1 || S < 1 || nb_cap < 1 || W < 1 || stride < 1 || shift < 0 || nscopes < 1 ||
        max_work < 0 || qstep < 16 || nrounds < 1 || round_stride < 0)
        return F3D_ERR_CONFIG;
    F3D_CUDA_TRY(f3d_launch(plan::plan_round_kernel, dim3(nrounds), dim3(plan::kThreads), 0,
                            (cudaStream_t)stream, counts, base, K, S, nb_cap, W, stride, 0,
                            shift % W, round_stride, nscopes, scope_seg, scope_nseg, seg_start,
                            seg_vstart, scope_len, scope_order, work, max_work, qstep, live));
    return F3D_OK;
}

extern "C" int f3d_plan_pool(const int32_t* counts, const int32_t* base, int nslots, int cap,
                             int rho, int32_t* tile_start, int32_t* tile_m, int32_t* tile_out,
                             int32_t* totals, void* stream) {
    if (nslots < 1 || cap < 1 || rho < 1) return F3D_ERR_CONFIG;
    plan::plan_pool_kernel<<<1, plan::kThreads, 0, (cudaStream_t)stream>>>(
        counts, base, nslots, cap, rho, tile_start, tile_m, tile_out, totals);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
