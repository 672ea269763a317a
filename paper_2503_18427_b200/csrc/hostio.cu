// Host <-> device transfers of dense row-major matrices for the handle tier
// (the reference-facing calls: aes_spmm_sampled, aes_gcn_forward, ..., and
// the pybind `_core` module over them).
//
// A caller's buffer is usually PAGEABLE (a numpy array).  cudaMemcpy from
// pageable memory is staged by the driver through a small pinned bounce
// buffer on one CPU thread, and a D2H copy into a freshly allocated numpy
// output also takes its first-touch page faults on that one thread: the
// products SpMM call moved 2.5 GB that way in ~380 ms (6.5 GB/s).  Here
// pageable buffers go through the library's own pinned staging ring
// (kStages x kChunk bytes) with the host side of every chunk copied by a
// small pool of CPU threads, overlapped with the DMA of the neighbouring
// chunks.  Pinned (registered / cudaMallocHost) buffers keep the direct
// cudaMemcpy2DAsync.  Results are byte-identical either way.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aes {
namespace {

constexpr size_t kChunk = 32u << 20;  // bytes per staging buffer
constexpr int kStages = 4;

// Fixed pool of worker threads running slices of a parallel_for.
class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return (int)workers_.size() + 1; }
    // fn(i) for i in [0, n), the calling thread takes part
    void run(int n, const std::function<void(int)>& fn) {
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            n_ = n;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return done_ == n_; });
        fn_ = nullptr;
    }

  private:
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* fn;
            {
                std::lock_guard<std::mutex> g(m_);
                if (!fn_ || next_ >= n_) return;
                i = next_++;
                fn = fn_;
            }
            (*fn)(i);
            std::lock_guard<std::mutex> g(m_);
            if (++done_ == n_) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

struct Stager {
    std::mutex m;  // one staged transfer at a time per process
    void* buf[kStages] = {};
    cudaEvent_t ev[kStages] = {};
    bool ready = false;
    Pool* pool = nullptr;
    int init() {
        if (ready) return AES_OK;
        for (int i = 0; i < kStages; ++i) {
            AES_CUDA_TRY(cudaHostAlloc(&buf[i], kChunk, cudaHostAllocDefault));
            AES_CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        const unsigned hc = std::thread::hardware_concurrency();
        pool = new Pool((int)std::min(15u, hc > 1 ? hc - 1 : 1u));
        ready = true;
        return AES_OK;
    }
};
Stager& stager() {
    static Stager* s = new Stager;  // never destroyed: process-lifetime pinned ring
    return *s;
}

bool pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// memcpy of `bytes` split over the pool (>= 1 MB per slice)
void par_copy(Pool* pool, void* dst, const void* src, size_t bytes) {
    const int slices = (int)std::max<size_t>(1, std::min<size_t>((size_t)pool->size(), bytes >> 20));
    const size_t per = (bytes + slices - 1) / slices;
    pool->run(slices, [&](int i) {
        const size_t o = (size_t)i * per;
        if (o < bytes) memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(per, bytes - o));
    });
}

}  // namespace

int h2d_dense(const float* h, uint64_t rows, uint64_t cols, float* d, uint64_t ld, cudaStream_t st) {
    if (rows == 0 || cols == 0) return AES_OK;
    const size_t row_bytes = cols * sizeof(float);
    if (!pageable(h) || rows * row_bytes < (4u << 20)) {
        AES_CUDA_TRY(cudaMemcpy2DAsync(d, ld * sizeof(float), h, row_bytes, row_bytes, rows, cudaMemcpyHostToDevice,
                                       st));
        return AES_OK;
    }
    Stager& s = stager();
    std::lock_guard<std::mutex> g(s.m);
    AES_TRY(s.init());
    const uint64_t rows_per = std::max<uint64_t>(1, kChunk / row_bytes);
    int k = 0;
    for (uint64_t r0 = 0; r0 < rows; r0 += rows_per, k = (k + 1) % kStages) {
        const uint64_t nr = std::min(rows_per, rows - r0);
        AES_CUDA_TRY(cudaEventSynchronize(s.ev[k]));  // this staging buffer's previous DMA is done
        par_copy(s.pool, s.buf[k], reinterpret_cast<const char*>(h) + r0 * row_bytes, nr * row_bytes);
        AES_CUDA_TRY(cudaMemcpy2DAsync(d + r0 * ld, ld * sizeof(float), s.buf[k], row_bytes, row_bytes, nr,
                                       cudaMemcpyHostToDevice, st));
        AES_CUDA_TRY(cudaEventRecord(s.ev[k], st));
    }
    return AES_OK;
}

int d2h_dense(const float* d, uint64_t ld, uint64_t rows, uint64_t cols, float* h, cudaStream_t st) {
    if (rows == 0 || cols == 0) return AES_OK;
    const size_t row_bytes = cols * sizeof(float);
    if (!pageable(h) || rows * row_bytes < (4u << 20)) {
        AES_CUDA_TRY(cudaMemcpy2DAsync(h, row_bytes, d, ld * sizeof(float), row_bytes, rows, cudaMemcpyDeviceToHost,
                                       st));
        return AES_OK;
    }
    Stager& s = stager();
    std::lock_guard<std::mutex> g(s.m);
    AES_TRY(s.init());
    const uint64_t rows_per = std::max<uint64_t>(1, kChunk / row_bytes);
    const uint64_t chunks = (rows + rows_per - 1) / rows_per;
    auto enqueue = [&](uint64_t c) -> int {
        const int k = (int)(c % kStages);
        const uint64_t r0 = c * rows_per, nr = std::min(rows_per, rows - r0);
        AES_CUDA_TRY(cudaMemcpy2DAsync(s.buf[k], row_bytes, d + r0 * ld, ld * sizeof(float), row_bytes, nr,
                                       cudaMemcpyDeviceToHost, st));
        AES_CUDA_TRY(cudaEventRecord(s.ev[k], st));
        return AES_OK;
    };
    // DMA runs kStages - 1 chunks ahead of the host copies out of the ring
    for (uint64_t c = 0; c < std::min<uint64_t>(chunks, kStages - 1); ++c) AES_TRY(enqueue(c));
    for (uint64_t c = 0; c < chunks; ++c) {
        if (c + kStages - 1 < chunks) AES_TRY(enqueue(c + kStages - 1));
        const int k = (int)(c % kStages);
        AES_CUDA_TRY(cudaEventSynchronize(s.ev[k]));
        const uint64_t r0 = c * rows_per, nr = std::min(rows_per, rows - r0);
        par_copy(s.pool, reinterpret_cast<char*>(h) + r0 * row_bytes, s.buf[k], nr * row_bytes);
    }
    return AES_OK;
}

}  // namespace aes
