// Adaptive edge sampler for sm_100a: per-row strategy (Table 1 / Eq. 3), a
// single-pass decoupled look-back scan building the sampled row pointer, and a
// slot-order fill producing the sampled CSR that the SpMM consumes.
//
// Reference: proj/src/sampling.cpp:29-152 (plans), proj/src/spmm.cpp:54-76
// (the per-row buffer fill, which here is materialised once per (graph, W)
// and reused by every layer), proj/src/matrix.cpp:28-63 (validate_csr,
// row_stats).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {

// ===========================================================================
// Row-count scan: out[0] = 0, out[i+1] = sum_{r<=i} count(r).
// One pass over row_ptr; tile prefixes chained with decoupled look-back.
// ===========================================================================
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanIters = 8;                        // rows per thread per tile
constexpr int kScanTile = kScanThreads * kScanIters; // 2048 rows per tile

// Row count of row r, with the row's offsets b = row_ptr[r], e = row_ptr[r+1]
// already at hand (the tile stages row_ptr in shared memory).
template <int KIND>
__device__ __forceinline__ uint64_t row_count(const ScanArgs& a, uint64_t r, uint64_t b, uint64_t e) {
    if (KIND == kScanExplicit) {  // host-supplied plans: slots = chunk * cnt
        const uint2 p = reinterpret_cast<const uint2*>(a.row_params)[r];
        return (uint64_t)p.x * p.y;
    }
    const uint64_t nnz = e - b;
    if (KIND == kScanSlots) {
        // slots = chunk * cnt is min(nnz, W) for Sfs / Afs, and for Adaptive
        // whenever W is a multiple of 32 (every Table-1 branch then has
        // chunk * cnt == W: W/4*4, W/8*8, W/16*16, W/32*32); nnz for Full
        if (!a.row_params && (a.strategy != AES_ADAPTIVE || a.width % 32 == 0))
            return a.strategy == AES_FULL ? nnz : min(nnz, (uint64_t)a.width);
        const RowParams p = row_params(nnz, a.width, a.strategy);
        if (a.row_params) reinterpret_cast<uint2*>(a.row_params)[r] = make_uint2(p.chunk, p.cnt);
        return (uint64_t)p.chunk * p.cnt;
    } else if (KIND == kScanStarts) {
        const RowParams p = row_params(nnz, a.width, a.strategy);
        return row_num_starts(nnz, a.width, a.strategy, p);
    } else {  // kScanGcnNnz: rows are sorted (validated); probe the diagonal
        if (!a.add_self_loops) return nnz;
        uint64_t lo = b, hi = e;
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (a.col_ind[mid] < r) lo = mid + 1; else hi = mid;
        }
        const bool has_diag = lo < e && a.col_ind[lo] == r;
        return nnz + (has_diag ? 0 : 1);
    }
}

// shared-memory index of tile row i: one u64 of padding per 16 so that the
// blocked per-thread reads (thread t: rows 8t..8t+7) spread over the banks
__device__ __forceinline__ int pad_idx(int i) { return i + (i >> 4); }

// Reduce-then-scan over 2048-row tiles, two kernels with no inter-CTA waits
// (a decoupled look-back measured latency-bound here: ~1 200 tiles chained
// through L2 round trips took 40 us for 39 MB).
//   pass 1  tile totals: tile_tot[t] = sum of the tile's row counts
//   pass 2  each tile sums the totals before it (<= a few thousand u64 from
//           L2, a block reduction), scans its rows and writes srow_ptr
// The tile's row_ptr (2049 values) is staged in shared memory with coalesced
// loads; thread t owns rows 8t..8t+7 (one thread-serial prefix, one block
// scan per tile); prefixes go back through shared memory so the srow_ptr
// stores are coalesced.
constexpr int kPadded = kScanTile + 1 + (kScanTile + 1) / 16 + 1;

template <int KIND>
__device__ __forceinline__ uint64_t tile_counts(const ScanArgs& a, uint64_t base, int nr, uint64_t* s_rp,
                                                uint64_t (&incl)[kScanIters], bool write_params) {
    const int tid = threadIdx.x;
    if (KIND != kScanExplicit)
        for (int i = tid; i <= nr; i += kScanThreads) s_rp[pad_idx(i)] = a.row_ptr[base + i];
    __syncthreads();
    ScanArgs aa = a;
    if (!write_params) aa.row_params = KIND == kScanExplicit ? a.row_params : nullptr;
    uint64_t run = 0;
#pragma unroll
    for (int u = 0; u < kScanIters; ++u) {
        const int i = tid * kScanIters + u;
        uint64_t c = 0;
        if (i < nr) {
            const uint64_t b = KIND != kScanExplicit ? s_rp[pad_idx(i)] : 0;
            const uint64_t e = KIND != kScanExplicit ? s_rp[pad_idx(i + 1)] : 0;
            c = row_count<KIND>(aa, base + i, b, e);
        }
        run += c;
        incl[u] = run;
    }
    return run;
}

// block-wide exclusive scan of one u64 per thread; *total gets the sum
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t* warp_tot, uint64_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) warp_tot[wid] = v;
    __syncthreads();
    uint64_t woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        const uint64_t y = warp_tot[w];
        woff += (w < wid) ? y : 0;
        tot += y;
    }
    *total = tot;
    return woff + v - x;
}

template <int KIND>
__global__ void __launch_bounds__(kScanThreads)
row_tile_total_kernel(ScanArgs a, unsigned long long* tile_tot) {
    __shared__ uint64_t s_rp[kPadded];
    __shared__ uint64_t warp_tot[kScanThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    const int nr = (int)min((uint64_t)kScanTile, a.n - base);
    uint64_t incl[kScanIters];
    const uint64_t run = tile_counts<KIND>(a, base, nr, s_rp, incl, false);
    uint64_t tot;
    block_excl_scan(run, warp_tot, &tot);
    if (threadIdx.x == 0) tile_tot[blockIdx.x] = tot;
}

template <int KIND>
__global__ void __launch_bounds__(kScanThreads)
row_scan_kernel(ScanArgs a, const unsigned long long* __restrict__ tile_tot) {
    __shared__ uint64_t s_rp[kPadded];
    __shared__ uint64_t warp_tot[kScanThreads / 32];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x;
    const uint64_t tile = blockIdx.x;
    const uint64_t base = tile * kScanTile;
    const int nr = (int)min((uint64_t)kScanTile, a.n - base);
    // exclusive offset of this tile: the totals of every tile before it
    uint64_t pre = 0;
    for (uint64_t t = tid; t < tile; t += kScanThreads) pre += tile_tot[t];
    uint64_t incl[kScanIters];
    const uint64_t run = tile_counts<KIND>(a, base, nr, s_rp, incl, true);
    uint64_t pre_tot, tile_sum;
    block_excl_scan(pre, warp_tot, &pre_tot);
    __syncthreads();  // warp_tot reused
    const uint64_t thread_excl = block_excl_scan(run, warp_tot, &tile_sum);
    const uint64_t excl = pre_tot + thread_excl;
    __syncthreads();  // every s_rp read is done
#pragma unroll
    for (int u = 0; u < kScanIters; ++u) s_rp[pad_idx(tid * kScanIters + u)] = excl + incl[u];
    __syncthreads();
    for (int i = tid; i < nr; i += kScanThreads) a.out[base + i + 1] = s_rp[pad_idx(i)];
    if (tile == 0 && tid == 0) a.out[0] = 0;
}

// One cooperative launch instead of two kernels: every CTA owns a contiguous
// run of tiles.  Phase 1 sums its tiles' row counts (row_ptr from HBM) and
// publishes the CTA total; a grid barrier (co-residency guaranteed by the
// cooperative launch); phase 2 sums the totals of the CTAs before it, then
// rescans its tiles (row_ptr now an L2 hit: 16 B per row of the graph) and
// writes srow_ptr.  Saves one launch and one HBM pass over row_ptr.
// Counts of the first kCoopKeep tiles stay in registers across the barrier
// (u32 per row: a row count is at most 2^32 - 1 for every kind but the
// caller-supplied explicit plans, which recount instead).
constexpr int kCoopKeep = 4;
template <int KIND>
__global__ void __launch_bounds__(kScanThreads, 4)
row_scan_coop_kernel(ScanArgs a, unsigned long long* cta_tot, unsigned int* barrier, uint32_t tiles_per_cta) {
    constexpr int K = KIND == kScanExplicit ? 0 : kCoopKeep;
    __shared__ uint64_t s_rp[kPadded];
    __shared__ uint64_t warp_tot[kScanThreads / 32];
    const int tid = threadIdx.x;
    const uint64_t n_tiles = (a.n + kScanTile - 1) / kScanTile;
    const uint64_t t0 = (uint64_t)blockIdx.x * tiles_per_cta;
    const uint64_t t1 = min(n_tiles, t0 + tiles_per_cta);
    uint32_t keep[K > 0 ? K : 1][kScanIters];
    uint64_t incl[kScanIters];
    uint64_t mine = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint64_t t = t0 + k;
        if (t < t1) {
            const uint64_t base = t * kScanTile;
            const int nr = (int)min((uint64_t)kScanTile, a.n - base);
            const uint64_t run = tile_counts<KIND>(a, base, nr, s_rp, incl, true);  // (params written once)
            uint64_t prev = 0;
#pragma unroll
            for (int u = 0; u < kScanIters; ++u) {
                keep[k][u] = (uint32_t)(incl[u] - prev);
                prev = incl[u];
            }
            mine += run;
            __syncthreads();  // s_rp reused by the next tile
        }
    }
    for (uint64_t t = t0 + K; t < t1; ++t) {
        const uint64_t base = t * kScanTile;
        const int nr = (int)min((uint64_t)kScanTile, a.n - base);
        mine += tile_counts<KIND>(a, base, nr, s_rp, incl, false);
        __syncthreads();
    }
    uint64_t cta_sum;
    block_excl_scan(mine, warp_tot, &cta_sum);
    if (tid == 0) {
        cta_tot[blockIdx.x] = cta_sum;
        __threadfence();
        atomicAdd(barrier, 1u);
        unsigned int seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(barrier) : "memory");
        } while (seen < gridDim.x);
    }
    __syncthreads();
    uint64_t pre = 0;
    for (uint32_t c = tid; c < blockIdx.x; c += kScanThreads) pre += __ldcg(cta_tot + c);
    uint64_t run_off;
    block_excl_scan(pre, warp_tot, &run_off);
    __syncthreads();  // warp_tot reused
    auto emit = [&](uint64_t t) {  // incl holds this thread's inclusive counts of tile t
        const uint64_t base = t * kScanTile;
        const int nr = (int)min((uint64_t)kScanTile, a.n - base);
        uint64_t tile_sum;
        const uint64_t excl = run_off + block_excl_scan(incl[kScanIters - 1], warp_tot, &tile_sum);
        __syncthreads();  // every s_rp / warp_tot read is done
#pragma unroll
        for (int u = 0; u < kScanIters; ++u) s_rp[pad_idx(tid * kScanIters + u)] = excl + incl[u];
        __syncthreads();
        for (int i = tid; i < nr; i += kScanThreads) a.out[base + i + 1] = s_rp[pad_idx(i)];
        run_off += tile_sum;
        __syncthreads();
    };
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (t0 + k < t1) {
            uint64_t r = 0;
#pragma unroll
            for (int u = 0; u < kScanIters; ++u) incl[u] = (r += keep[k][u]);
            emit(t0 + k);
        }
    for (uint64_t t = t0 + K; t < t1; ++t) {
        const uint64_t base = t * kScanTile;
        const int nr = (int)min((uint64_t)kScanTile, a.n - base);
        tile_counts<KIND>(a, base, nr, s_rp, incl, true);
        __syncthreads();
        emit(t);
    }
    if (blockIdx.x == 0 && tid == 0) a.out[0] = 0;
}

template <int KIND>
int launch_scan_kind(const ScanArgs& a, void* ws, cudaStream_t st) {
    const uint64_t tiles = (a.n + kScanTile - 1) / kScanTile;
    auto* hdr = reinterpret_cast<unsigned int*>(ws);
    auto* tot = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
    static int occ_dev[kMaxDevices] = {};
    int& occ = occ_dev[cur_device()];
    if (occ == 0) {
        AES_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, row_scan_coop_kernel<KIND>, kScanThreads, 0));
        if (occ < 1) occ = -1;
    }
    if (tiles > 1 && occ > 0) {
        // kCoopKeep tiles per CTA when the grid fits (counts never recomputed)
        const uint64_t slots = (uint64_t)num_sms() * occ;
        const uint32_t per = (uint32_t)((tiles + slots - 1) / slots);
        const unsigned grid = (unsigned)((tiles + per - 1) / per);
        AES_CUDA_TRY(cudaMemsetAsync(hdr, 0, sizeof(unsigned int), st));
        ScanArgs aa = a;
        unsigned long long* tp = tot;
        unsigned int* bp = hdr;
        uint32_t pp = per;
        void* args[] = {&aa, &tp, &bp, &pp};
        if (cudaLaunchCooperativeKernel((const void*)row_scan_coop_kernel<KIND>, dim3(grid), dim3(kScanThreads),
                                        args, 0, st) == cudaSuccess)
            return AES_OK;
        (void)cudaGetLastError();  // not launchable cooperatively here: the two-kernel form
    }
    row_tile_total_kernel<KIND><<<(unsigned)tiles, kScanThreads, 0, st>>>(a, tot);
    row_scan_kernel<KIND><<<(unsigned)tiles, kScanThreads, 0, st>>>(a, tot);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace

size_t row_scan_workspace_bytes(uint64_t n) {
    uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 0) tiles = 1;
    return 256 + tiles * sizeof(unsigned long long);
}

int launch_row_scan(int kind, const ScanArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
    size_t need = row_scan_workspace_bytes(a.n);
    if (ws == nullptr || ws_bytes < need) return fail(AES_ERR_INVALID_ARG, "scan workspace too small");
    if (a.n == 0) {
        AES_CUDA_TRY(cudaMemsetAsync(a.out, 0, sizeof(uint64_t), st));
        return AES_OK;
    }
    switch (kind) {
        case kScanSlots: return launch_scan_kind<kScanSlots>(a, ws, st);
        case kScanStarts: return launch_scan_kind<kScanStarts>(a, ws, st);
        case kScanExplicit: return launch_scan_kind<kScanExplicit>(a, ws, st);
        default: return launch_scan_kind<kScanGcnNnz>(a, ws, st);
    }
}

// ===========================================================================
// Slot-order fill.  A CTA owns 256 consecutive rows and flattens their slots;
// each thread takes slots in stride, finds its row by binary search over the
// sampled row pointer staged in shared memory, and copies one (col, val) —
// writes are fully coalesced, reads are contiguous runs of chunk_len.
// ===========================================================================
namespace {

constexpr int kFillRows = 256;
constexpr int kFillMap = 8192;  // slots per pass of the slot -> row map (u8 entries)

// Per-row fill parameters, computed once per row (not per slot).
struct FillRow {
    uint64_t src;     // row_ptr[row] of the matrix being filled
    uint32_t first;   // first slot, relative to the CTA's first slot
    uint32_t cnt;     // sample_cnt
    uint32_t shift;   // log2(cnt) when cnt is a power of two, else 0xff
    uint32_t range;   // hash modulus nnz - chunk + 1 (adaptive, sampled rows), saturated to 2^32-1
    uint32_t mode;    // 0: start 0 (whole row / prefix), 1: hashed windows, 2: AFS starts
    uint32_t nnz;     // plan row nnz (AFS)
};

// The CTA owns kFillRows consecutive rows and writes their slots in slot
// order (coalesced scol / sval stores; each window's reads are contiguous).
// Thread i derives row i's parameters once and writes i into the slot -> row
// map for the row's slots, so a slot finds its row with one shared load (no
// search); the slot's window index s and offset j come from a shift/mask
// (sample_cnt is a power of two in every Table-1 branch when W >= 32), and a
// hashed start needs at most a 32-bit modulo: s*1429 < 32*1429, and
// hash_start is s*1429 itself whenever the modulus exceeds it.  CTAs whose
// slots exceed the map (W > 32, FULL) run several passes.
constexpr int kFillUnroll = 4;  // slots per thread per step, all loads in flight before the stores
__global__ void __launch_bounds__(kFillRows, 6)
sample_fill_kernel(const uint64_t* __restrict__ plan_row_ptr, const uint64_t* __restrict__ row_ptr,
                   const uint32_t* __restrict__ col_ind, const float* __restrict__ val,
                   uint64_t n, uint32_t width, int strategy, const uint64_t* __restrict__ srow_ptr,
                   uint32_t* __restrict__ scol, float* __restrict__ sval) {
    __shared__ FillRow s_row[kFillRows];
    __shared__ unsigned char s_map[kFillMap];
    __shared__ uint64_t s_first[kFillRows + 1];
    const int tid = threadIdx.x;
    const uint64_t r0 = (uint64_t)blockIdx.x * kFillRows;
    const int nr = (int)min((uint64_t)kFillRows, n - r0);
    // one round of independent loads per row (no dependent load chain before
    // the map is built): sampled offsets, plan row length, source row start
    uint64_t my_s0 = 0, my_nnz = 0, my_src = 0;
    if (tid < nr) {
        const uint64_t r = r0 + tid;
        my_s0 = srow_ptr[r];
        my_nnz = plan_row_ptr[r + 1] - plan_row_ptr[r];
        my_src = row_ptr[r];
        s_first[tid] = my_s0;
        if (tid == nr - 1) s_first[nr] = srow_ptr[r + 1];
    }
    __syncthreads();
    const uint64_t g0 = s_first[0], total = s_first[nr] - g0;
    uint32_t my_first = 0, my_slots = 0;
    if (tid < nr) {
        const uint64_t nnz = my_nnz;
        const RowParams p = row_params(nnz, width, strategy);
        FillRow fr;
        fr.src = my_src;
        my_first = (uint32_t)(my_s0 - g0);
        my_slots = p.chunk * p.cnt;
        fr.first = my_first;
        fr.cnt = p.cnt;
        fr.shift = (p.cnt && (p.cnt & (p.cnt - 1)) == 0) ? (uint32_t)__ffs(p.cnt) - 1 : 0xffu;
        fr.nnz = (uint32_t)nnz;
        if (strategy == AES_AFS) {
            fr.mode = 2;
        } else if (strategy == AES_ADAPTIVE && nnz > width) {
            fr.mode = 1;
        } else {
            fr.mode = 0;
        }
        const uint64_t range = nnz - (uint64_t)p.chunk + 1ull;
        fr.range = range > 0xffffffffull ? 0xffffffffu : (uint32_t)range;
        s_row[tid] = fr;
    }
    // (total < 2^32 slots per CTA: 256 rows of u32 nonzeros each at most)
    for (uint32_t pass = 0; pass < total; pass += kFillMap) {
        const uint32_t pend = (uint32_t)min((uint64_t)pass + kFillMap, total);
        __syncthreads();  // previous pass done with the map
        if (tid < nr && my_slots) {
            const uint32_t a = max(my_first, pass), b = min(my_first + my_slots, pend);
            for (uint32_t t = a; t < b; ++t) s_map[t - pass] = (unsigned char)tid;
        }
        __syncthreads();
        // kFillUnroll slots per thread per step: their loads are all in
        // flight before the first store (the map / row lookups are
        // shared-memory hits)
        for (uint32_t t0 = pass + tid; t0 < pend; t0 += kFillUnroll * kFillRows) {
            uint64_t src[kFillUnroll];
            bool ok[kFillUnroll];
#pragma unroll
            for (int u = 0; u < kFillUnroll; ++u) {
                const uint32_t t = t0 + u * kFillRows;
                ok[u] = t < pend;
                src[u] = 0;
                if (ok[u]) {
                    const FillRow& fr = s_row[s_map[t - pass]];
                    const uint32_t k = t - fr.first;
                    uint32_t sidx, j;
                    if (fr.shift != 0xffu) {
                        sidx = k & (fr.cnt - 1);
                        j = k >> fr.shift;
                    } else {
                        sidx = k % fr.cnt;
                        j = k / fr.cnt;
                    }
                    uint32_t start = 0;
                    if (fr.mode == 1) {
                        const uint32_t prod = sidx * 1429u;  // sidx < cnt <= 32 on hashed rows
                        start = prod < fr.range ? prod : prod % fr.range;
                    } else if (fr.mode == 2) {
                        start = (uint32_t)((uint64_t)sidx * fr.nnz / fr.cnt);
                    }
                    src[u] = fr.src + start + j;
                }
            }
            uint32_t cv[kFillUnroll];
            float vv[kFillUnroll];
#pragma unroll
            for (int u = 0; u < kFillUnroll; ++u)
                if (ok[u]) {
                    cv[u] = __ldg(col_ind + src[u]);
                    vv[u] = __ldg(val + src[u]);
                }
#pragma unroll
            for (int u = 0; u < kFillUnroll; ++u)
                if (ok[u]) {
                    const uint64_t pos = g0 + t0 + u * kFillRows;
                    __stcs(scol + pos, cv[u]);
                    __stcs(sval + pos, vv[u]);
                }
        }
    }
}

// Fill from host-supplied plans (RowSamplePlan objects built outside
// build_plan_set): chunk/cnt per row as uint2, starts in CSR form.  Same slot
// order as spmm.cpp:68-76.
__global__ void __launch_bounds__(kFillRows)
explicit_fill_kernel(const uint64_t* __restrict__ row_ptr, const uint2* __restrict__ params,
                     const uint64_t* __restrict__ starts_ptr, const uint32_t* __restrict__ starts,
                     const uint32_t* __restrict__ col_ind, const float* __restrict__ val, uint64_t n,
                     const uint64_t* __restrict__ srow_ptr, uint32_t* __restrict__ scol, float* __restrict__ sval) {
    __shared__ uint64_t s_srow[kFillRows + 1];
    const uint64_t r0 = (uint64_t)blockIdx.x * kFillRows;
    const int nr = (int)min((uint64_t)kFillRows, n - r0);
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_srow[i] = srow_ptr[r0 + i];
    __syncthreads();
    const uint64_t g0 = s_srow[0];
    const uint64_t total = s_srow[nr] - g0;
    for (uint64_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint64_t pos = g0 + t;
        int lo = 0, hi = nr;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (s_srow[mid] <= pos) lo = mid; else hi = mid;
        }
        const uint64_t row = r0 + lo;
        const uint2 p = params[row];
        const uint64_t k = pos - s_srow[lo];
        const uint64_t s = k % p.y, j = k / p.y;
        const uint64_t src = row_ptr[row] + starts[starts_ptr[row] + s] + j;
        scol[pos] = col_ind[src];
        sval[pos] = val[src];
    }
}

// Coverage of explicit plans (sampling_rate's unique count, sampling.cpp:136-147):
// mark every sampled offset, then count marks per matrix.
__global__ void explicit_mark_kernel(const uint64_t* __restrict__ row_ptr, const uint2* __restrict__ params,
                                     const uint64_t* __restrict__ starts_ptr, const uint32_t* __restrict__ starts,
                                     uint64_t n, unsigned char* __restrict__ seen) {
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint2 p = params[r];
        const uint64_t slots = (uint64_t)p.x * p.y;
        const uint64_t sp = starts_ptr[r], base = row_ptr[r];
        for (uint64_t k = lane; k < slots; k += 32) {
            const uint64_t s = k % p.y, j = k / p.y;
            seen[base + starts[sp + s] + j] = 1;
        }
    }
}

__global__ void count_marks_kernel(const unsigned char* __restrict__ seen, uint64_t nnz,
                                   unsigned long long* __restrict__ total) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz; i += (uint64_t)gridDim.x * blockDim.x)
        c += seen[i];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(total, c);
}

__global__ void explicit_slots_kernel(const uint64_t* __restrict__ row_ptr, const uint2* __restrict__ params,
                                      uint64_t n, double* __restrict__ per_row, unsigned long long* __restrict__ totals) {
    unsigned long long slots = 0, nnz_sum = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t nnz = row_ptr[r + 1] - row_ptr[r];
        const uint2 p = params[r];
        nnz_sum += nnz;
        if (nnz == 0) {
            if (per_row) per_row[r] = 1.0;
            continue;
        }
        const uint64_t sl = (uint64_t)p.x * p.y;
        slots += sl;
        if (per_row) per_row[r] = (double)sl / (double)nnz;
    }
    for (int o = 16; o > 0; o >>= 1) {
        slots += __shfl_down_sync(0xffffffffu, slots, o);
        nnz_sum += __shfl_down_sync(0xffffffffu, nnz_sum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&totals[0], slots);
        atomicAdd(&totals[2], nnz_sum);
    }
}

// Export RowSamplePlan data (module.cpp:72-81) as flat arrays.
__global__ void plan_export_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n, uint32_t width,
                                   int strategy, const uint64_t* __restrict__ starts_ptr,
                                   uint32_t* __restrict__ chunk, uint32_t* __restrict__ cnt,
                                   uint32_t* __restrict__ starts) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t nnz = row_ptr[r + 1] - row_ptr[r];
        RowParams p = row_params(nnz, width, strategy);
        chunk[r] = p.chunk;
        cnt[r] = p.cnt;
        uint32_t ns = row_num_starts(nnz, width, strategy, p);
        uint64_t b = starts_ptr[r];
        for (uint32_t s = 0; s < ns; ++s) starts[b + s] = row_start(nnz, width, strategy, p, s);
    }
}

// sampling_rate (sampling.cpp:120-152): per-row slots/nnz, and totals of
// slots, distinct sampled offsets and nnz (integer sums -> deterministic).
__global__ void sampling_rate_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n, uint32_t width,
                                     int strategy, double* __restrict__ per_row,
                                     unsigned long long* __restrict__ totals) {
    uint64_t slots_sum = 0, uniq_sum = 0, nnz_sum = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t nnz = row_ptr[r + 1] - row_ptr[r];
        nnz_sum += nnz;
        if (nnz == 0) {
            if (per_row) per_row[r] = 1.0;
            continue;
        }
        RowParams p = row_params(nnz, width, strategy);
        uint64_t slots = (uint64_t)p.chunk * p.cnt;
        slots_sum += slots;
        if (per_row) per_row[r] = (double)slots / (double)nnz;
        uint64_t uniq;
        if (strategy == AES_FULL) {
            uniq = nnz;
        } else if (strategy == AES_SFS) {
            uniq = p.chunk;
        } else if (strategy == AES_AFS) {
            uniq = p.cnt;  // floor(s*nnz/cnt) strictly increases for cnt <= nnz
        } else if (nnz <= width) {
            uniq = nnz;
        } else {
            // union of cnt (<= 32) windows of length chunk
            uint32_t st[32];
            uint32_t c = p.cnt;
            for (uint32_t s = 0; s < c; ++s) st[s] = hash_start(s, nnz, p.chunk);
            for (uint32_t i = 1; i < c; ++i) {  // insertion sort
                uint32_t v = st[i];
                int j = (int)i - 1;
                while (j >= 0 && st[j] > v) { st[j + 1] = st[j]; --j; }
                st[j + 1] = v;
            }
            uniq = 0;
            uint64_t cover_end = 0;  // exclusive end of covered prefix
            for (uint32_t s = 0; s < c; ++s) {
                uint64_t b = st[s], e = b + p.chunk;
                if (b < cover_end) b = cover_end;
                if (e > b) { uniq += e - b; cover_end = e; }
            }
        }
        uniq_sum += uniq;
    }
    for (int o = 16; o > 0; o >>= 1) {
        slots_sum += __shfl_down_sync(0xffffffffu, slots_sum, o);
        uniq_sum += __shfl_down_sync(0xffffffffu, uniq_sum, o);
        nnz_sum += __shfl_down_sync(0xffffffffu, nnz_sum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&totals[0], (unsigned long long)slots_sum);
        atomicAdd(&totals[1], (unsigned long long)uniq_sum);
        atomicAdd(&totals[2], (unsigned long long)nnz_sum);
    }
}

// row_stats (matrix.cpp:54-63)
__global__ void row_stats_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n,
                                 uint64_t* __restrict__ row_nnz, unsigned long long* __restrict__ max_nnz) {
    unsigned long long m = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t d = row_ptr[r + 1] - row_ptr[r];
        if (row_nnz) row_nnz[r] = d;
        m = d > m ? d : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_down_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(max_nnz, m);
}

// validate_csr (matrix.cpp:28-52), pass 1: first decreasing row_ptr step.
__global__ void validate_monotonic_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n,
                                          unsigned long long* __restrict__ first_bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (row_ptr[i + 1] < row_ptr[i]) atomicMin(first_bad, (unsigned long long)(i + 1));
    }
}

// pass 2: warp per row; the first offending element of the lowest row wins.
// code = (row << 2) | error, error 2 = ColumnOutOfRange, 3 = UnsortedRow.
__global__ void validate_rows_kernel(const uint64_t* __restrict__ row_ptr,
                                     const uint32_t* __restrict__ col, uint64_t n, uint64_t n_cols,
                                     unsigned long long* __restrict__ first_bad) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t b = row_ptr[r], e = row_ptr[r + 1];
        for (uint64_t k0 = b; k0 < e; k0 += 32) {
            uint64_t k = k0 + lane;
            int err = 0;
            if (k < e) {
                uint32_t c = col[k];
                if (c >= n_cols) err = AES_CSR_COL_OUT_OF_RANGE;
                else if (k > b && c <= col[k - 1]) err = AES_CSR_UNSORTED;
            }
            unsigned bad = __ballot_sync(0xffffffffu, err != 0);
            if (bad) {
                int first = __ffs(bad) - 1;
                int e_first = __shfl_sync(0xffffffffu, err, first);
                if (lane == 0) atomicMin(first_bad, (unsigned long long)((r << 2) | (uint64_t)e_first));
                break;
            }
        }
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Internal launchers used by the handle API
// ---------------------------------------------------------------------------
int launch_sample_fill(const uint64_t* plan_row_ptr, const uint64_t* row_ptr, const uint32_t* col,
                       const float* val, uint64_t n, uint32_t width, int strategy,
                       const uint64_t* srow_ptr, uint32_t* scol, float* sval, cudaStream_t st) {
    if (n == 0) return AES_OK;
    unsigned grid = grid_for(n, kFillRows);
    sample_fill_kernel<<<grid, kFillRows, 0, st>>>(plan_row_ptr, row_ptr, col, val, n, width, strategy,
                                                   srow_ptr, scol, sval);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

// Caller-built plans (aes_plan_from_host) are checked before any fill or
// mark reads through them: every window s of row r must satisfy
// start_s + chunk <= row_nnz (or chunk == 0), the only reads the reference
// makes (spmm.cpp:68-76).  The smallest offending row is recorded.
__global__ void explicit_check_kernel(const uint64_t* __restrict__ row_ptr, const uint2* __restrict__ params,
                                      const uint64_t* __restrict__ starts_ptr, const uint32_t* __restrict__ starts,
                                      uint64_t n, unsigned long long* __restrict__ bad_row) {
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint2 p = params[r];
        if (p.x == 0) continue;
        const uint64_t nnz = row_ptr[r + 1] - row_ptr[r];
        const uint64_t sp = starts_ptr[r];
        bool bad = false;
        for (uint32_t s = lane; s < p.y; s += 32) bad |= (uint64_t)starts[sp + s] + p.x > nnz;
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(bad_row, (unsigned long long)r);
    }
}

int launch_explicit_check(const uint64_t* row_ptr, const uint32_t* params, const uint64_t* starts_ptr,
                          const uint32_t* starts, uint64_t n, unsigned long long* bad_row, cudaStream_t st) {
    AES_CUDA_TRY(cudaMemsetAsync(bad_row, 0xff, sizeof(unsigned long long), st));
    if (n == 0) return AES_OK;
    explicit_check_kernel<<<grid_for(n * 32, 256, num_sms() * 32), 256, 0, st>>>(
        row_ptr, reinterpret_cast<const uint2*>(params), starts_ptr, starts, n, bad_row);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_explicit_fill(const uint64_t* row_ptr, const uint32_t* params, const uint64_t* starts_ptr,
                         const uint32_t* starts, const uint32_t* col, const float* val, uint64_t n,
                         const uint64_t* srow_ptr, uint32_t* scol, float* sval, cudaStream_t st) {
    if (n == 0) return AES_OK;
    explicit_fill_kernel<<<grid_for(n, kFillRows), kFillRows, 0, st>>>(
        row_ptr, reinterpret_cast<const uint2*>(params), starts_ptr, starts, col, val, n, srow_ptr, scol, sval);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_explicit_rate(const uint64_t* row_ptr, const uint32_t* params, const uint64_t* starts_ptr,
                         const uint32_t* starts, uint64_t n, uint64_t nnz, unsigned char* seen, double* per_row,
                         unsigned long long* totals, cudaStream_t st) {
    AES_CUDA_TRY(cudaMemsetAsync(totals, 0, 3 * sizeof(unsigned long long), st));
    if (n == 0) return AES_OK;
    const uint2* pp = reinterpret_cast<const uint2*>(params);
    explicit_slots_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(row_ptr, pp, n, per_row, totals);
    if (nnz) {
        AES_CUDA_TRY(cudaMemsetAsync(seen, 0, nnz, st));
        explicit_mark_kernel<<<grid_for(n * 32, 256, num_sms() * 32), 256, 0, st>>>(row_ptr, pp, starts_ptr, starts, n, seen);
        count_marks_kernel<<<grid_for(nnz, 256, num_sms() * 16), 256, 0, st>>>(seen, nnz, totals + 1);
    }
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_plan_export(const uint64_t* row_ptr, uint64_t n, uint32_t width, int strategy,
                       const uint64_t* starts_ptr, uint32_t* chunk, uint32_t* cnt, uint32_t* starts,
                       cudaStream_t st) {
    if (n == 0) return AES_OK;
    plan_export_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(row_ptr, n, width, strategy,
                                                                   starts_ptr, chunk, cnt, starts);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_sampling_rate(const uint64_t* row_ptr, uint64_t n, uint32_t width, int strategy,
                         double* per_row, unsigned long long* totals, cudaStream_t st) {
    AES_CUDA_TRY(cudaMemsetAsync(totals, 0, 3 * sizeof(unsigned long long), st));
    if (n == 0) return AES_OK;
    sampling_rate_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(row_ptr, n, width, strategy,
                                                                     per_row, totals);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_row_stats(const uint64_t* row_ptr, uint64_t n, uint64_t* row_nnz,
                     unsigned long long* max_nnz, cudaStream_t st) {
    AES_CUDA_TRY(cudaMemsetAsync(max_nnz, 0, sizeof(unsigned long long), st));
    if (n == 0) return AES_OK;
    row_stats_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(row_ptr, n, row_nnz, max_nnz);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_validate(const uint64_t* row_ptr, const uint32_t* col, uint64_t n, uint64_t n_cols,
                    unsigned long long* scratch2, cudaStream_t st) {
    AES_CUDA_TRY(cudaMemsetAsync(scratch2, 0xff, 2 * sizeof(unsigned long long), st));
    if (n == 0) return AES_OK;
    validate_monotonic_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(row_ptr, n, scratch2);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_validate_rows(const uint64_t* row_ptr, const uint32_t* col, uint64_t n, uint64_t n_cols,
                         unsigned long long* scratch, cudaStream_t st) {
    if (n == 0) return AES_OK;
    validate_rows_kernel<<<grid_for(n * 32, 256, num_sms() * 32), 256, 0, st>>>(row_ptr, col, n, n_cols,
                                                                         scratch);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace aes

// ===========================================================================
// C ABI: device tier
// ===========================================================================
extern "C" {

size_t aes_dev_scan_workspace_bytes(uint64_t n_rows) {
    size_t a = aes::row_scan_workspace_bytes(n_rows);
    size_t b = 256 + 2 * 148 * 8 * 32;  // fit_params partials
    return a > b ? a : b;
}

int aes_dev_sample_plan(const uint64_t* plan_row_ptr, uint64_t n_rows, uint32_t width, int strategy,
                        uint64_t* srow_ptr, uint32_t* row_params, void* workspace,
                        size_t workspace_bytes, void* stream) {
    if (width == 0) return aes::fail(AES_ERR_ZERO_WIDTH, "ZeroWidth");
    if (strategy < 0 || strategy > 3) return aes::fail(AES_ERR_INVALID_ARG, "unknown strategy");
    aes::ScanArgs a{plan_row_ptr, nullptr, n_rows, width, strategy, 0, srow_ptr, row_params};
    return aes::launch_row_scan(aes::kScanSlots, a, workspace, workspace_bytes, aes::as_stream(stream));
}

int aes_dev_sample_fill(const uint64_t* plan_row_ptr, const uint64_t* row_ptr,
                        const uint32_t* col_ind, const float* val, uint64_t n_rows, uint32_t width,
                        int strategy, const uint64_t* srow_ptr, uint32_t* scol, float* sval,
                        void* stream) {
    if (width == 0) return aes::fail(AES_ERR_ZERO_WIDTH, "ZeroWidth");
    return aes::launch_sample_fill(plan_row_ptr, row_ptr, col_ind, val, n_rows, width, strategy,
                                   srow_ptr, scol, sval, aes::as_stream(stream));
}

}  // extern "C"
