// Row-sharded GCN forward with an NCCL all-gather per layer: the C-ABI form
// of gcn.ShardedGCN(exchange="nccl") for C / C++ callers that own an
// ncclComm_t (aes_gcn_forward_sharded(..., ncclComm_t);
// reference semantics: gcn_forward, proj/src/gnn.cpp:66-78).
//
// Each rank holds its contiguous equal-size row shard of the sampled CSR
// (absolute slot offsets, a view of the global plan) and a full replica of
// the layer input.  Per layer: sampled SpMM of the shard rows -> ordered-fp32
// GEMM + bias (+ ReLU) into a [rows_per_rank, round4(fout)] send block ->
// ncclAllGather of the blocks, in rank order, into the other replica, which
// the next layer reads with row stride round4(fout): the exchange moves
// N * round4(fout) * 4 bytes, not N * ld * 4 (a 40-wide class layer in a
// 128-wide replica would otherwise move 3.2x the bytes).  The
// concatenation equals the single-GPU layer output bit for bit (plans are
// per-row independent).
//
// NCCL is resolved at run time from the process's own libnccl.so.2 (the one
// that created `comm`; torch's bundled copy when torch is loaded), so the
// library has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <mutex>

#include "common.cuh"

namespace aes {
namespace {

typedef ncclResult_t (*AllGatherFn)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
typedef const char* (*ErrStrFn)(ncclResult_t);
typedef ncclResult_t (*AsyncErrFn)(ncclComm_t, ncclResult_t*);

struct NcclApi {
    AllGatherFn all_gather = nullptr;
    ErrStrFn err_str = nullptr;
    AsyncErrFn async_err = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.all_gather = reinterpret_cast<AllGatherFn>(dlsym(h, "ncclAllGather"));
        api.err_str = reinterpret_cast<ErrStrFn>(dlsym(h, "ncclGetErrorString"));
        api.async_err = reinterpret_cast<AsyncErrFn>(dlsym(h, "ncclCommGetAsyncError"));
    });
    return api;
}

constexpr uint64_t round4(uint64_t x) { return (x + 3) & ~3ull; }

}  // namespace
}  // namespace aes

extern "C" {

uint64_t aes_gcn_sharded_workspace_bytes(uint64_t rows_per_rank, uint64_t ld) {
    return 2 * rows_per_rank * aes::round4(ld) * sizeof(float) + 256;
}

int aes_gcn_forward_sharded(const uint64_t* srow_shard, const uint32_t* scol, const float* sval, uint64_t shard_rows,
                            uint64_t rows_per_rank, int n_layers, const uint64_t* dims, const float* const* weights,
                            const float* const* biases, int finite_w, float* replica_a, float* replica_b, uint64_t ld,
                            uint64_t max_row_slots, void* workspace, size_t workspace_bytes, void* nccl_comm,
                            float** out_replica, uint64_t* out_ld, void* stream) {
    using namespace aes;
    if (n_layers < 1 || !dims || !weights || !replica_a || !replica_b || !out_replica || !nccl_comm)
        return fail(AES_ERR_INVALID_ARG, "null argument");
    if (shard_rows > rows_per_rank) return fail(AES_ERR_INVALID_ARG, "shard_rows > rows_per_rank");
    if (ld % 4 != 0) return fail(AES_ERR_INVALID_ARG, "replica ld must be a multiple of 4");
    for (int l = 0; l <= n_layers; ++l)
        if (dims[l] == 0 || dims[l] > ld) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    if (workspace_bytes < aes_gcn_sharded_workspace_bytes(rows_per_rank, ld) || !workspace)
        return fail(AES_ERR_INVALID_ARG, "sharded GCN workspace too small");
    const NcclApi& nccl = nccl_api();
    if (!nccl.all_gather) return fail(AES_ERR_UNSUPPORTED, "libnccl.so.2 not found");
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
    cudaStream_t st = as_stream(stream);
    float* agg = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(workspace) + 127) & ~uintptr_t(127));
    float* send = agg + rows_per_rank * ld;
    // padding rows / columns of the send block hold zeros (finite values
    // are all the next SpMM's pad lanes ever see)
    AES_CUDA_TRY(cudaMemsetAsync(send, 0, rows_per_rank * ld * sizeof(float), st));
    float* in = replica_a;
    float* next = replica_b;
    uint64_t ld_in = ld;  // layer 0 reads the caller's replica layout
    for (int l = 0; l < n_layers; ++l) {
        const uint64_t fin = dims[l], fout = dims[l + 1];
        const uint64_t ld_out = round4(fout);  // compact next-layer replica
        if (shard_rows) {
            AES_TRY(aes_dev_spmm_f32_ex(srow_shard, scol, sval, shard_rows, in, ld_in, fin, agg, ld, max_row_slots,
                                        st));
            float* dst = send;
            AES_TRY(aes_dev_gemm_bias_act_ex(agg, shard_rows, fin, ld, weights[l], fout, fout,
                                             biases ? biases[l] : nullptr, l + 1 < n_layers, finite_w, &dst, nullptr,
                                             1, 0, ld_out, st));
        }
        const ncclResult_t r = nccl.all_gather(send, next, rows_per_rank * ld_out, ncclFloat32, comm, st);
        if (r != ncclSuccess)
            return fail(AES_ERR_CUDA, std::string("ncclAllGather: ") + (nccl.err_str ? nccl.err_str(r) : "error"));
        if (nccl.async_err) {  // a peer failure surfaces here, not as a hang later
            ncclResult_t ar = ncclSuccess;
            if (nccl.async_err(comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
                return fail(AES_ERR_CUDA, std::string("NCCL async error: ") + (nccl.err_str ? nccl.err_str(ar) : "error"));
        }
        float* t = in;
        in = next;
        next = t;
        ld_in = ld_out;
    }
    *out_replica = in;
    if (out_ld) *out_ld = ld_in;
    return AES_OK;
}

}  // extern "C"
