// Binary graph / feature files straight into HBM.
//
// Formats are the reference's (proj/src/io.cpp:117-220, proj/include/aesspmm/io.hpp):
//   CSRB: "CSRB", u8 version=1, u64 n_rows, u64 n_cols, u64 nnz,
//         u64 row_ptr[n+1], u32 col_ind[nnz], f32 val[nnz]
//   FMAT: "FMAT", u8 version=1, u8 dtype (0 = f32, 1 = u8 codes), u64 rows,
//         u64 cols, [dtype 1: f32 x_min, f32 x_max], payload row-major
// The payload is streamed file -> pinned staging (two 64 MB buffers) -> HBM
// with the read of chunk i+1 overlapping the H2D copy of chunk i, so an int8
// FMAT (a quarter of the f32 bytes) loads ~4x faster — the paper's feature-
// loading reduction.  int8 files become HBM-resident
// QuantizedFeatures (codes + exact LUT) with no host-side dequantization.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <unistd.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aes {
// defined in capi.cu
void* capi_alloc(size_t bytes);
void capi_free(void* p);
int capi_make_qfeat_u8(const uint8_t* d_codes, uint64_t rows, uint64_t cols, uint64_t ld, float lo, float hi,
                       aes_qfeat_t* out);
int capi_csr_from_device(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, uint64_t* rp, uint32_t* col, float* val,
                         aes_csr_t* out);
int capi_qfeat_device(aes_qfeat_t q, const void** codes, uint64_t* ld, int* u8);
int capi_csr_device(aes_csr_t a, const uint64_t** rp, const uint32_t** col, const float** val, uint64_t* n_rows,
                    uint64_t* n_cols, uint64_t* nnz);

namespace {

constexpr size_t kChunk = 64ull << 20;

struct Staging {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    std::mutex mu;
    int init() {
        if (buf[0]) return AES_OK;
        for (int i = 0; i < 2; ++i) {
            AES_CUDA_TRY(cudaMallocHost(&buf[i], kChunk));
            AES_CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
        AES_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        return AES_OK;
    }
};
Staging& staging() {  // per device: the staging stream and events belong to one device
    static Staging s[kMaxDevices];
    return s[cur_device()];
}

// Drains the staging stream on every exit path of stream_rows, so an error
// return never leaves a DMA still writing into a buffer the caller frees.
struct DrainGuard {
    cudaStream_t st;
    ~DrainGuard() {
        if (st) cudaStreamSynchronize(st);
    }
};

struct File {
    FILE* f = nullptr;
    std::string path;
    ~File() {
        if (f) fclose(f);
    }
};

int io_fail(const std::string& what, const std::string& path) { return fail(AES_ERR_IO, what + ": " + path); }

template <typename T>
int read_pod(File& fh, T* v) {
    if (fread(v, sizeof(T), 1, fh.f) != 1) return io_fail("TruncatedFile", fh.path);
    return AES_OK;
}

int open_magic(File& fh, const char* path, const char magic[4]) {
    fh.path = path;
    fh.f = fopen(path, "rb");
    if (!fh.f) return io_fail("Io: cannot open for reading", path);
    char m[4];
    if (fread(m, 1, 4, fh.f) != 4 || memcmp(m, magic, 4) != 0) return io_fail("BadMagic", path);
    uint8_t version = 0;
    AES_TRY(read_pod(fh, &version));
    if (version != 1) return io_fail(std::string("unsupported ") + std::string(magic, 4) + " version", path);
    return AES_OK;
}

// Read `bytes` at file offset `pos` with several threads (page-cache copies
// are memcpy-bound on one core; the pinned buffer then goes out by DMA).
bool parallel_pread(int fd, char* dst, uint64_t bytes, int64_t pos) {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned nt = bytes < (8u << 20) ? 1u : (hw > 16 ? 16u : (hw ? hw : 1u));
    const uint64_t per = (bytes + nt - 1) / nt;
    std::atomic<bool> ok{true};
    auto work = [&](unsigned t) {
        uint64_t off = t * per, end = off + per < bytes ? off + per : bytes;
        while (off < end) {
            ssize_t r = pread(fd, dst + off, end - off, pos + (int64_t)off);
            if (r <= 0) {
                ok = false;
                return;
            }
            off += (uint64_t)r;
        }
    };
    if (nt == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& x : th) x.join();
    }
    return ok;
}

// Stream `rows` rows of `row_bytes` from the file into dst (row pitch
// dst_pitch bytes), double-buffered through pinned memory.  zero_pitch:
// clear the whole destination (row padding included) first, ordered before
// the copies on the same stream.
int stream_rows(File& fh, void* dst, uint64_t rows, uint64_t row_bytes, uint64_t dst_pitch, bool zero_pitch = false) {
    if (rows == 0 || row_bytes == 0) return AES_OK;
    Staging& s = staging();
    std::lock_guard<std::mutex> lock(s.mu);
    AES_TRY(s.init());
    DrainGuard drain{s.st};
    if (zero_pitch) AES_CUDA_TRY(cudaMemsetAsync(dst, 0, rows * dst_pitch, s.st));
    const uint64_t rows_per = row_bytes >= kChunk ? 1 : kChunk / row_bytes;
    if (row_bytes > kChunk) return io_fail("row larger than the staging chunk", fh.path);
    int b = 0;
    const int fd = fileno(fh.f);
    int64_t pos = ftell(fh.f);
    for (uint64_t r0 = 0; r0 < rows; r0 += rows_per, b ^= 1) {
        const uint64_t nr = rows - r0 < rows_per ? rows - r0 : rows_per;
        AES_CUDA_TRY(cudaEventSynchronize(s.done[b]));  // this buffer's previous copy has drained
        if (!parallel_pread(fd, static_cast<char*>(s.buf[b]), nr * row_bytes, pos))
            return io_fail("TruncatedFile", fh.path);
        pos += (int64_t)(nr * row_bytes);
        AES_CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dst_pitch, dst_pitch, s.buf[b], row_bytes,
                                       row_bytes, nr, cudaMemcpyHostToDevice, s.st));
        AES_CUDA_TRY(cudaEventRecord(s.done[b], s.st));
    }
    AES_CUDA_TRY(cudaStreamSynchronize(s.st));
    fseek(fh.f, pos, SEEK_SET);  // keep the FILE position in step for the next array
    return AES_OK;
}

// A flat array of `bytes` from the file into dst, in staging-sized chunks.
int stream_bytes(File& fh, void* dst, uint64_t bytes) {
    for (uint64_t off = 0; off < bytes; off += kChunk) {
        const uint64_t nb = bytes - off < kChunk ? bytes - off : kChunk;
        AES_TRY(stream_rows(fh, static_cast<char*>(dst) + off, 1, nb, nb));
    }
    return AES_OK;
}

int write_all(FILE* f, const void* p, size_t n, const std::string& path) {
    if (n && fwrite(p, 1, n, f) != n) return io_fail("Io: write failed", path);
    return AES_OK;
}

struct FmatHeader {
    uint8_t dtype = 0;
    uint64_t rows = 0, cols = 0;
    float lo = 0.f, hi = 0.f;
};

int read_fmat_header(File& fh, const char* path, FmatHeader& h) {
    AES_TRY(open_magic(fh, path, "FMAT"));
    AES_TRY(read_pod(fh, &h.dtype));
    AES_TRY(read_pod(fh, &h.rows));
    AES_TRY(read_pod(fh, &h.cols));
    if (h.dtype == 1) {
        AES_TRY(read_pod(fh, &h.lo));
        AES_TRY(read_pod(fh, &h.hi));
    } else if (h.dtype != 0) {
        return io_fail("UnsupportedDtype", path);
    }
    return AES_OK;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace aes

extern "C" {

int aes_fmat_info(const char* path, int* dtype, uint64_t* rows, uint64_t* cols, float* x_min, float* x_max) {
    using namespace aes;
    File fh;
    FmatHeader h;
    AES_TRY(read_fmat_header(fh, path, h));
    if (dtype) *dtype = h.dtype;
    if (rows) *rows = h.rows;
    if (cols) *cols = h.cols;
    if (x_min) *x_min = h.lo;
    if (x_max) *x_max = h.hi;
    return AES_OK;
}

int aes_fmat_load_device(const char* path, void* d_dst, uint64_t ld_elems, double* load_ms) {
    using namespace aes;
    auto t0 = std::chrono::steady_clock::now();
    File fh;
    FmatHeader h;
    AES_TRY(read_fmat_header(fh, path, h));
    const uint64_t esz = h.dtype == 0 ? 4 : 1;
    if (ld_elems < h.cols) return fail(AES_ERR_INVALID_ARG, "leading dimension smaller than the file's columns");
    AES_TRY(stream_rows(fh, d_dst, h.rows, h.cols * esz, ld_elems * esz));
    if (load_ms) *load_ms = ms_since(t0);
    return AES_OK;
}

int aes_fmat_load_qfeat(const char* path, aes_qfeat_t* out, double* load_ms) {
    using namespace aes;
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    auto t0 = std::chrono::steady_clock::now();
    File fh;
    FmatHeader h;
    AES_TRY(read_fmat_header(fh, path, h));
    if (h.dtype != 1) return io_fail("FMAT dtype 1 (u8 codes) expected", path);
    const uint64_t ld = (h.cols + 15) & ~15ull;  // 16-B code rows (int8 SpMM batch kernel)
    auto* codes = static_cast<uint8_t*>(capi_alloc(h.rows * ld + 16));
    if (!codes) return fail(AES_ERR_CUDA, "alloc");
    int s = stream_rows(fh, codes, h.rows, h.cols, ld, ld != h.cols);
    if (!s) s = capi_make_qfeat_u8(codes, h.rows, h.cols, ld, h.lo, h.hi, out);  // takes ownership
    if (s) {
        capi_free(codes);
        return s;
    }
    if (load_ms) *load_ms = ms_since(t0);
    return AES_OK;
}

int aes_fmat_save_f32(const float* x, uint64_t rows, uint64_t cols, const char* path) {
    using namespace aes;
    FILE* f = fopen(path, "wb");
    if (!f) return io_fail("Io: cannot open for writing", path);
    uint8_t version = 1, dtype = 0;
    int s = write_all(f, "FMAT", 4, path);
    if (!s) s = write_all(f, &version, 1, path);
    if (!s) s = write_all(f, &dtype, 1, path);
    if (!s) s = write_all(f, &rows, 8, path);
    if (!s) s = write_all(f, &cols, 8, path);
    if (!s) s = write_all(f, x, rows * cols * 4, path);
    fclose(f);
    return s;
}

int aes_fmat_save_qfeat(aes_qfeat_t q, const char* path) {
    using namespace aes;
    uint64_t rows = 0, cols = 0;
    float lo = 0, hi = 0;
    uint32_t bits = 0;
    AES_TRY(aes_qfeat_info(q, &rows, &cols, &lo, &hi, &bits));
    if (bits != 8) return fail(AES_ERR_INVALID_ARG, "FMAT dtype 1 stores 8-bit codes only");  // io.cpp:167-169
    const void* codes = nullptr;
    uint64_t ld = 0;
    int u8 = 0;
    AES_TRY(capi_qfeat_device(q, &codes, &ld, &u8));
    if (!u8) return fail(AES_ERR_INVALID_ARG, "FMAT dtype 1 stores 8-bit codes only");
    std::string host(rows * cols, '\0');
    if (rows * cols)
        AES_CUDA_TRY(cudaMemcpy2D(&host[0], cols, codes, ld, cols, rows, cudaMemcpyDeviceToHost));
    FILE* f = fopen(path, "wb");
    if (!f) return io_fail("Io: cannot open for writing", path);
    uint8_t version = 1, dtype = 1;
    int s = write_all(f, "FMAT", 4, path);
    if (!s) s = write_all(f, &version, 1, path);
    if (!s) s = write_all(f, &dtype, 1, path);
    if (!s) s = write_all(f, &rows, 8, path);
    if (!s) s = write_all(f, &cols, 8, path);
    if (!s) s = write_all(f, &lo, 4, path);
    if (!s) s = write_all(f, &hi, 4, path);
    if (!s) s = write_all(f, host.data(), host.size(), path);
    fclose(f);
    return s;
}

int aes_csr_load(const char* path, aes_csr_t* out, double* load_ms) {
    using namespace aes;
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    auto t0 = std::chrono::steady_clock::now();
    File fh;
    AES_TRY(open_magic(fh, path, "CSRB"));
    uint64_t n = 0, m = 0, nnz = 0;
    AES_TRY(read_pod(fh, &n));
    AES_TRY(read_pod(fh, &m));
    AES_TRY(read_pod(fh, &nnz));
    auto* rp = static_cast<uint64_t*>(capi_alloc((n + 1) * 8));
    auto* col = static_cast<uint32_t*>(capi_alloc((nnz ? nnz : 1) * 4));
    auto* val = static_cast<float*>(capi_alloc((nnz ? nnz : 1) * 4));
    int s = (rp && col && val) ? AES_OK : fail(AES_ERR_CUDA, "alloc");
    if (!s) s = stream_bytes(fh, rp, (n + 1) * 8);
    if (!s) s = stream_bytes(fh, col, nnz * 4);
    if (!s) s = stream_bytes(fh, val, nnz * 4);
    // validate_csr on the GPU (io.cpp:142-143): "invalid CSR payload: <message>"
    if (!s) s = capi_csr_from_device(n, m, nnz, rp, col, val, out);
    if (s) {
        capi_free(rp);
        capi_free(col);
        capi_free(val);
        if (s == AES_ERR_CSR_INVALID) return io_fail(std::string("invalid CSR payload: ") + aes_last_error(), path);
        return s;
    }
    if (load_ms) *load_ms = ms_since(t0);
    return AES_OK;
}

int aes_csr_save(aes_csr_t a, const char* path) {
    using namespace aes;
    const uint64_t* rp;
    const uint32_t* col;
    const float* val;
    uint64_t n, m, nnz;
    AES_TRY(capi_csr_device(a, &rp, &col, &val, &n, &m, &nnz));
    std::string buf((n + 1) * 8 + nnz * 8, '\0');
    AES_CUDA_TRY(cudaMemcpy(&buf[0], rp, (n + 1) * 8, cudaMemcpyDeviceToHost));
    if (nnz) {
        AES_CUDA_TRY(cudaMemcpy(&buf[(n + 1) * 8], col, nnz * 4, cudaMemcpyDeviceToHost));
        AES_CUDA_TRY(cudaMemcpy(&buf[(n + 1) * 8 + nnz * 4], val, nnz * 4, cudaMemcpyDeviceToHost));
    }
    FILE* f = fopen(path, "wb");
    if (!f) return io_fail("Io: cannot open for writing", path);
    uint8_t version = 1;
    int s = write_all(f, "CSRB", 4, path);
    if (!s) s = write_all(f, &version, 1, path);
    if (!s) s = write_all(f, &n, 8, path);
    if (!s) s = write_all(f, &m, 8, path);
    if (!s) s = write_all(f, &nnz, 8, path);
    if (!s) s = write_all(f, buf.data(), buf.size(), path);
    fclose(f);
    return s;
}

}  // extern "C"
