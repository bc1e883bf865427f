// Host-buffer entry points: the reference's numpy signatures one-to-one (KN:84, 103, 135-136) --
// host pointers in, planes mutated in place, counts out.  These are what a `meshlayers._native`
// stub binds directly.
//
// The reference's call shape makes the caller's planes live in pageable host memory, so a naive
// twin moves every plane over PCIe twice (round 1: 1.76 GB and 143 ms for one raster_tea at
// 16384^2, 12 GB/s effective).  Three things change that here:
//
//   1. A persistent ARENA per process: one device region (grown on demand, bump-allocated per call),
//      four pinned 16 MiB staging chunks, two streams, a small worker pool.  No cudaMalloc /
//      cudaFree, no pageable-memory DMA inside a call.
//   2. Pipelined uploads: the worker pool copies chunk k+1 of a pageable array into pinned staging
//      while chunk k is on the wire.  float32 triangle arrays travel as float32.
//   3. SPARSE WRITE-BACK.  coverage_fill and raster_tea only ever SET texels (out = 1 resp.
//      data = value, mask = 1, edited = 1; KN:97-99, 198-202) and count how many target bytes were 0.
//      The kernels therefore run against a ZEROED device scratch plane -- nothing of the caller's
//      planes is uploaded -- which afterwards holds exactly the set of texels written.  The set comes
//      back as 1 bit per texel, or as the list of its non-zero 64-texel words when that is smaller,
//      and the host applies the reference's write rule to its own planes (worker pool, rows of the
//      caller's memory), counting 0 -> 1 transitions there.  PCIe traffic per stroke: the triangle
//      arrays up, O(hit texels / 8) bytes down, instead of 6 plane transfers.
//
// raster_depth needs the caller's depth values on the device (min with the existing plane), but its
// plane is window sized (4 MB at 1024^2); it uses the arena and the pipelined upload.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include "internal.h"

namespace {

#define ML_TRY(call) do { int _rc = (call); if (_rc != ML_OK) return _rc; } while (0)

// ------------------------------------------------------------------------------------------------
// worker pool: run(n, fn) calls fn(0..n-1) on the pool's threads and the caller, returns when done
class Pool {
public:
    explicit Pool(int n) : n_(n) {
        for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        { std::lock_guard<std::mutex> g(m_); stop_ = true; ++gen_; }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return n_ + 1; }
    void run(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1 || n_ == 0) { for (int i = 0; i < parts; ++i) fn(i); return; }
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn; parts_ = parts; next_ = 0; pending_ = n_; ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }
private:
    void work() {
        for (;;) {
            int i;
            { std::lock_guard<std::mutex> g(m_); if (next_ >= parts_) return; i = next_++; }
            (*fn_)(i);
        }
    }
    void loop(int) {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            work();
            { std::lock_guard<std::mutex> g(m_); if (--pending_ == 0) done_.notify_one(); }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int parts_ = 0, next_ = 0, pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

void par_memcpy(Pool& pool, void* dst, const void* src, size_t bytes) {
    const size_t grain = 2u << 20;
    if (bytes < 2 * grain) { memcpy(dst, src, bytes); return; }
    const int parts = (int)std::min<size_t>((bytes + grain - 1) / grain, (size_t)pool.size() * 2);
    const size_t per = ((bytes + parts - 1) / parts + 63) & ~(size_t)63;
    pool.run(parts, [&](int i) {
        const size_t a = (size_t)i * per;
        if (a < bytes) memcpy((char*)dst + a, (const char*)src + a, std::min(per, bytes - a));
    });
}

// ------------------------------------------------------------------------------------------------
constexpr size_t PIN_CHUNK = 16u << 20;
constexpr int NPIN = 4;

struct Arena {
    std::mutex mu;                      // one host-plane call at a time (the reference's single-writer rule)
    int device = -1;
    char* base = nullptr;
    size_t cap = 0, off = 0;
    char* pin[NPIN] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t pin_ev[NPIN] = {nullptr, nullptr, nullptr, nullptr};
    bool pin_busy[NPIN] = {false, false, false, false};
    int pin_next = 0;
    cudaStream_t s_up = nullptr, s_run = nullptr;
    cudaEvent_t ev = nullptr;
    Pool* pool = nullptr;

    int init() {
        int dev = 0;
        ML_CUDA(cudaGetDevice(&dev));
        if (device == dev && pool) return ML_OK;
        if (device != -1 && device != dev) release();
        device = dev;
        ML_CUDA(cudaStreamCreateWithFlags(&s_up, cudaStreamNonBlocking));
        ML_CUDA(cudaStreamCreateWithFlags(&s_run, cudaStreamNonBlocking));
        ML_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        for (int i = 0; i < NPIN; ++i) {
            ML_CUDA(cudaHostAlloc((void**)&pin[i], PIN_CHUNK, cudaHostAllocDefault));
            ML_CUDA(cudaEventCreateWithFlags(&pin_ev[i], cudaEventDisableTiming));
            pin_busy[i] = false;
        }
        unsigned hc = std::thread::hardware_concurrency();
        int workers = hc > 2 ? (int)std::min(hc / 2, 8u) - 1 : 0;
        if (const char* e = getenv("ML_HOST_THREADS")) workers = std::max(0, atoi(e) - 1);
        pool = new Pool(workers);
        return ML_OK;
    }
    void release() {
        if (pool) { delete pool; pool = nullptr; }
        if (base) { cudaFree(base); base = nullptr; cap = 0; }
        for (int i = 0; i < NPIN; ++i) {
            if (pin[i]) { cudaFreeHost(pin[i]); pin[i] = nullptr; }
            if (pin_ev[i]) { cudaEventDestroy(pin_ev[i]); pin_ev[i] = nullptr; }
        }
        if (s_up) { cudaStreamDestroy(s_up); s_up = nullptr; }
        if (s_run) { cudaStreamDestroy(s_run); s_run = nullptr; }
        if (ev) { cudaEventDestroy(ev); ev = nullptr; }
        device = -1;
    }
    // start a call that needs `bytes` of device scratch in total
    int begin(size_t bytes) {
        ML_TRY(init());
        if (bytes > cap) {
            if (base) { ML_CUDA(cudaDeviceSynchronize()); ML_CUDA(cudaFree(base)); base = nullptr; cap = 0; }
            const size_t want = (bytes + (bytes >> 3) + ((size_t)1 << 20)) & ~(((size_t)1 << 20) - 1);
            ML_CUDA(cudaMalloc((void**)&base, want));
            cap = want;
        }
        off = 0;
        return ML_OK;
    }
    template <typename T> T* take(size_t bytes) {
        char* p = base + off;
        off += (bytes + 255) & ~(size_t)255;
        return (T*)p;
    }
    static size_t padded(size_t bytes) { return (bytes + 255) & ~(size_t)255; }

    int slot(int* out) {                // next pinned chunk, free for the host to write / read
        const int k = pin_next;
        pin_next = (pin_next + 1) % NPIN;
        if (pin_busy[k]) { ML_CUDA(cudaEventSynchronize(pin_ev[k])); pin_busy[k] = false; }
        *out = k;
        return ML_OK;
    }
    // pageable host -> device, staged through the pinned chunks; the pool fills chunk k+1 while chunk k flies
    int upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
        for (size_t a = 0; a < bytes; a += PIN_CHUNK) {
            const size_t len = std::min(PIN_CHUNK, bytes - a);
            int k = 0;
            ML_TRY(slot(&k));
            par_memcpy(*pool, pin[k], (const char*)src + a, len);
            ML_CUDA(cudaMemcpyAsync((char*)dst + a, pin[k], len, cudaMemcpyHostToDevice, st));
            ML_CUDA(cudaEventRecord(pin_ev[k], st));
            pin_busy[k] = true;
        }
        return ML_OK;
    }
    // device -> host consumer: `use(ptr, first_byte, len)` sees every chunk in pinned memory, the next chunk
    // is already on the wire while it runs
    int download(const void* src, size_t bytes, cudaStream_t st, const std::function<void(const char*, size_t, size_t)>& use) {
        struct Pending { int k; size_t a, len; };
        Pending q[NPIN];
        int qn = 0, qh = 0;
        size_t a = 0;
        auto issue = [&]() -> int {
            const size_t len = std::min(PIN_CHUNK, bytes - a);
            int k = 0;
            ML_TRY(slot(&k));
            ML_CUDA(cudaMemcpyAsync(pin[k], (const char*)src + a, len, cudaMemcpyDeviceToHost, st));
            ML_CUDA(cudaEventRecord(pin_ev[k], st));
            pin_busy[k] = true;
            q[(qh + qn) % NPIN] = Pending{k, a, len};
            ++qn;
            a += len;
            return ML_OK;
        };
        while (a < bytes && qn < 2) ML_TRY(issue());
        while (qn) {
            const Pending p = q[qh];
            qh = (qh + 1) % NPIN; --qn;
            ML_CUDA(cudaEventSynchronize(pin_ev[p.k]));
            pin_busy[p.k] = false;
            if (a < bytes) ML_TRY(issue());          // keep one transfer in flight while the host works on p
            use(pin[p.k], p.a, p.len);
        }
        return ML_OK;
    }
};

Arena g_arena;

// ML_HOST_TRACE=1: phase times of the host-buffer calls on stderr (each phase ends with a stream sync, so the
// traced call is slower than the untraced one; for finding out where a call spends its time)
struct Trace {
    bool on;
    double t0;
    static double now() { timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6; }
    Trace() : on(getenv("ML_HOST_TRACE") != nullptr), t0(now()) {}
    void mark(const char* what, cudaStream_t a = nullptr, cudaStream_t b = nullptr) {
        if (!on) return;
        if (a) cudaStreamSynchronize(a);
        if (b) cudaStreamSynchronize(b);
        const double t = now();
        fprintf(stderr, "[ml host] %-28s %7.3f ms\n", what, t - t0);
        t0 = t;
    }
};

// ------------------------------------------------------------------------------------------------
// device side of the sparse write-back: byte plane (0 / non-zero) -> 1 bit per texel, 64 texels per word,
// texel i = bit (i & 63) of word i >> 6; *nz += number of non-zero words.  plane is padded to a multiple of 64.
__global__ void __launch_bounds__(256)
pack64_kernel(const uint8_t* __restrict__ plane, long long nwords, unsigned long long* __restrict__ bits,
              unsigned long long* nz) {
    long long cnt = 0;
    const long long nthreads = (long long)gridDim.x * 256;
    for (long long w = (long long)blockIdx.x * 256 + threadIdx.x; w < nwords; w += nthreads) {
        const uint4* p = (const uint4*)(plane + (w << 6));
        unsigned long long word = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 v = ld_stream(p + k);
            const unsigned long long b16 = (unsigned long long)(nz_bits4(v.x) | (nz_bits4(v.y) << 4) | (nz_bits4(v.z) << 8) | (nz_bits4(v.w) << 12));
            word |= b16 << (16 * k);
        }
        bits[w] = word;
        cnt += word != 0;
    }
    block_count_add(cnt, nz);
}

// non-zero words -> list of (word index, bits) pairs, any order
__global__ void __launch_bounds__(256)
compact64_kernel(const unsigned long long* __restrict__ bits, long long nwords, unsigned long long* __restrict__ list,
                 unsigned long long* count) {
    const int lane = threadIdx.x & 31;
    const long long nthreads = (long long)gridDim.x * 256;
    for (long long w0 = (long long)blockIdx.x * 256; w0 < nwords; w0 += nthreads) {
        const long long w = w0 + threadIdx.x;
        const unsigned long long word = w < nwords ? bits[w] : 0ull;
        const unsigned bal = __ballot_sync(0xffffffffu, word != 0);
        if (!bal) continue;
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(count, (unsigned long long)__popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (word) {
            const unsigned long long at = slot + __popc(bal & ((1u << lane) - 1u));
            list[2 * at] = (unsigned long long)w;
            list[2 * at + 1] = word;
        }
    }
}

unsigned grid_for_words(long long nwords) {
    long long b = (nwords + 255) / 256;
    const long long cap = (long long)ml_sm_count() * 16;
    return (unsigned)std::max(1ll, std::min(b, cap));
}

// ------------------------------------------------------------------------------------------------
// host side: apply the reference's write rule to the caller's planes for the texels of one 64-texel word.
// Returns how many target bytes were 0 (KN:97 / KN:198).  data == NULL: coverage_fill (only `flag` is written).
template <int ES>
inline long long apply_word(unsigned long long word, long long i0, long long n, uint8_t* flag, uint8_t* mask, void* data,
                            uint32_t value) {
    long long newly = 0;
    if (word == ~0ull && i0 + 64 <= n) {                   // fully hit word: straight-line stores
        for (int b = 0; b < 64; ++b) newly += flag[i0 + b] == 0;
        memset(flag + i0, 1, 64);
        if (mask) memset(mask + i0, 1, 64);
        if (data) {
            if (ES == 1) memset((uint8_t*)data + i0, (int)(value & 0xffu), 64);
            else if (ES == 2) { uint16_t* d = (uint16_t*)data + i0; for (int b = 0; b < 64; ++b) d[b] = (uint16_t)value; }
            else { uint32_t* d = (uint32_t*)data + i0; for (int b = 0; b < 64; ++b) d[b] = value; }
        }
        return newly;
    }
    while (word) {
        const int b = __builtin_ctzll(word);
        word &= word - 1;
        const long long i = i0 + b;
        if (i >= n) break;
        newly += flag[i] == 0;
        flag[i] = 1;
        if (mask) mask[i] = 1;
        if (data) {
            if (ES == 1) ((uint8_t*)data)[i] = (uint8_t)value;
            else if (ES == 2) ((uint16_t*)data)[i] = (uint16_t)value;
            else ((uint32_t*)data)[i] = value;
        }
    }
    return newly;
}

long long apply_words(Pool& pool, const unsigned long long* words, long long first_word, long long nw, long long n,
                      uint8_t* flag, uint8_t* mask, void* data, int esize, uint32_t value) {
    const int parts = (int)std::max<long long>(1, std::min<long long>(pool.size() * 4, nw / 4096));
    std::vector<long long> acc((size_t)parts, 0);
    pool.run(parts, [&](int p) {
        const long long a = nw * p / parts, b = nw * (p + 1) / parts;
        long long c = 0;
        for (long long k = a; k < b; ++k) {
            const unsigned long long w = words[k];
            if (!w) continue;
            const long long i0 = (first_word + k) << 6;
            c += esize == 1 ? apply_word<1>(w, i0, n, flag, mask, data, value)
               : esize == 2 ? apply_word<2>(w, i0, n, flag, mask, data, value) : apply_word<4>(w, i0, n, flag, mask, data, value);
        }
        acc[(size_t)p] = c;
    });
    long long t = 0;
    for (long long c : acc) t += c;
    return t;
}

long long apply_list(Pool& pool, const unsigned long long* pairs, long long npairs, long long n,
                     uint8_t* flag, uint8_t* mask, void* data, int esize, uint32_t value) {
    const int parts = (int)std::max<long long>(1, std::min<long long>(pool.size() * 4, npairs / 1024));
    std::vector<long long> acc((size_t)parts, 0);
    pool.run(parts, [&](int p) {
        const long long a = npairs * p / parts, b = npairs * (p + 1) / parts;
        long long c = 0;
        for (long long k = a; k < b; ++k) {
            const long long i0 = (long long)pairs[2 * k] << 6;
            const unsigned long long w = pairs[2 * k + 1];
            c += esize == 1 ? apply_word<1>(w, i0, n, flag, mask, data, value)
               : esize == 2 ? apply_word<2>(w, i0, n, flag, mask, data, value) : apply_word<4>(w, i0, n, flag, mask, data, value);
        }
        acc[(size_t)p] = c;
    });
    long long t = 0;
    for (long long c : acc) t += c;
    return t;
}

// The set of texels a kernel wrote into the zeroed scratch plane `hit` (n texels, padded to 64) -> the caller's
// planes.  ctr[2] receives the non-zero word count; returns the number of `flag` bytes that were 0.
int write_back(Arena& A, const uint8_t* hit, long long n, unsigned long long* d_bits, unsigned long long* d_list,
               unsigned long long* d_ctr /* [4]: kernel counters [0], [1]; [2] nz words, [3] list count */,
               unsigned long long* ctr_out /* host copy of d_ctr[0..3] after the kernel */, uint8_t* flag, uint8_t* mask,
               void* data, int esize, uint32_t value, long long* newly) {
    const long long nwords = (n + 63) >> 6;
    pack64_kernel<<<grid_for_words(nwords), 256, 0, A.s_run>>>(hit, nwords, d_bits, d_ctr + 2);
    ML_CUDA(cudaGetLastError());
    int k = 0;
    ML_TRY(A.slot(&k));
    unsigned long long* c = (unsigned long long*)A.pin[k];
    ML_CUDA(cudaMemcpyAsync(c, d_ctr, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, A.s_run));
    ML_CUDA(cudaStreamSynchronize(A.s_run));
    for (int j = 0; j < 4; ++j) ctr_out[j] = c[j];
    const long long nz = (long long)c[2];
    *newly = 0;
    if (nz == 0) return ML_OK;
    long long total = 0;
    if (nz * 16 < nwords * 8 / 2) {
        // sparse: the non-zero words only
        compact64_kernel<<<grid_for_words(nwords), 256, 0, A.s_run>>>(d_bits, nwords, d_list, d_ctr + 3);
        ML_CUDA(cudaGetLastError());
        ML_TRY(A.download(d_list, (size_t)nz * 16, A.s_run, [&](const char* p, size_t, size_t len) {
            total += apply_list(*A.pool, (const unsigned long long*)p, (long long)(len / 16), n, flag, mask, data, esize, value);
        }));
    } else {
        ML_TRY(A.download(d_bits, (size_t)nwords * 8, A.s_run, [&](const char* p, size_t first, size_t len) {
            total += apply_words(*A.pool, (const unsigned long long*)p, (long long)(first / 8), (long long)(len / 8), n, flag, mask,
                                 data, esize, value);
        }));
    }
    *newly = total;
    return ML_OK;
}

size_t tri_elem(int tri_dtype) { return tri_dtype == ML_F32 ? sizeof(float) : sizeof(double); }

}  // namespace

extern "C" {

void ml_host_release(void) {
    std::lock_guard<std::mutex> g(g_arena.mu);
    g_arena.release();
}

int ml_coverage_fill_host(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                          uint8_t* out, int64_t* written) {
    if (written) *written = 0;
    if (width <= 0 || height <= 0 || ntri <= 0) return ML_OK;
    if (tri_dtype != ML_F32 && tri_dtype != ML_F64) return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    if (ml_sm_count() <= 0) return ml_fail(ML_ERR_NO_DEVICE, "no CUDA device");
    Arena& A = g_arena;
    std::lock_guard<std::mutex> g(A.mu);
    const long long n = (long long)width * height, nwords = (n + 63) >> 6;
    const size_t tri_bytes = (size_t)ntri * 6 * tri_elem(tri_dtype), ws = ml_raster_workspace_bytes(ntri);
    ML_TRY(A.begin(Arena::padded(tri_bytes) + Arena::padded((size_t)nwords * 64) + 2 * Arena::padded((size_t)nwords * 8) +
                   Arena::padded(ws) + 1024));
    void* d_tri = A.take<void>(tri_bytes);
    uint8_t* d_hit = A.take<uint8_t>((size_t)nwords * 64);
    unsigned long long* d_bits = A.take<unsigned long long>((size_t)nwords * 8);
    unsigned long long* d_list = A.take<unsigned long long>((size_t)nwords * 8);
    void* d_ws = A.take<void>(ws);
    unsigned long long* d_ctr = A.take<unsigned long long>(64);
    ML_CUDA(cudaMemsetAsync(d_hit, 0, (size_t)nwords * 64, A.s_run));
    ML_CUDA(cudaMemsetAsync(d_ctr, 0, 64, A.s_run));
    ML_TRY(A.upload(d_tri, tri_xy, tri_bytes, A.s_up));
    ML_CUDA(cudaEventRecord(A.ev, A.s_up));
    ML_CUDA(cudaStreamWaitEvent(A.s_run, A.ev, 0));
    ML_TRY(ml_coverage_fill(d_tri, tri_dtype, ntri, width, height, 0, height, d_hit, (uint64_t*)d_ctr, d_ws, ws, A.s_run));
    long long newly = 0;
    unsigned long long c[4];
    ML_TRY(write_back(A, d_hit, n, d_bits, d_list, d_ctr, c, out, nullptr, nullptr, 1, 1u, &newly));
    if (written) *written = newly;
    return ML_OK;
}

int ml_raster_depth_host(const void* tri_xy, const void* tri_zn, int tri_dtype, int64_t ntri,
                         float* depth, int64_t width, int64_t height, int64_t* updated) {
    if (updated) *updated = 0;
    if (width <= 0 || height <= 0 || ntri <= 0) return ML_OK;
    if (tri_dtype != ML_F32 && tri_dtype != ML_F64) return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    if (ml_sm_count() <= 0) return ml_fail(ML_ERR_NO_DEVICE, "no CUDA device");
    Arena& A = g_arena;
    std::lock_guard<std::mutex> g(A.mu);
    const size_t es = tri_elem(tri_dtype), plane = (size_t)width * height * sizeof(float), ws = ml_raster_workspace_bytes(ntri);
    ML_TRY(A.begin(Arena::padded((size_t)ntri * 6 * es) + Arena::padded((size_t)ntri * 3 * es) + Arena::padded(plane) + Arena::padded(ws)));
    void* d_tri = A.take<void>((size_t)ntri * 6 * es);
    void* d_zn = A.take<void>((size_t)ntri * 3 * es);
    float* d_depth = A.take<float>(plane);
    void* d_ws = A.take<void>(ws);
    ML_TRY(A.upload(d_depth, depth, plane, A.s_up));
    ML_TRY(A.upload(d_tri, tri_xy, (size_t)ntri * 6 * es, A.s_up));
    ML_TRY(A.upload(d_zn, tri_zn, (size_t)ntri * 3 * es, A.s_up));
    ML_CUDA(cudaEventRecord(A.ev, A.s_up));
    ML_CUDA(cudaStreamWaitEvent(A.s_run, A.ev, 0));
    ML_TRY(ml_raster_depth(d_tri, d_zn, tri_dtype, ntri, d_depth, width, height, d_ws, ws, A.s_run));
    // the reference's count is order dependent; report texels whose value changed
    long long changed = 0;
    ML_TRY(A.download(d_depth, plane, A.s_run, [&](const char* p, size_t first, size_t len) {
        const uint32_t* now = (const uint32_t*)p;
        uint32_t* old = (uint32_t*)((char*)depth + first);
        const size_t m = len / sizeof(float);
        for (size_t i = 0; i < m; ++i) { changed += now[i] != old[i]; old[i] = now[i]; }
    }));
    if (updated) *updated = changed;
    return ML_OK;
}

int ml_raster_tea_host(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri,
                       double ww, double wh, const float* depth, int64_t depth_w, int64_t depth_h,
                       double eps, int eps_f32, double sfx, double sfy, double bx, double by,
                       const uint8_t* shape, int64_t shape_w, int64_t shape_h,
                       void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                       int64_t width, int64_t height, int64_t* edited_count, int64_t* fragments) {
    if (edited_count) *edited_count = 0;
    if (fragments) *fragments = 0;
    if (width <= 0 || height <= 0 || ntri <= 0) return ML_OK;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (tri_dtype != ML_F32 && tri_dtype != ML_F64) return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    if (!(depth_w >= ceil(ww) && depth_h >= ceil(wh)))
        return ml_fail(ML_ERR_ARG, "depth plane smaller than the window");
    if (shape_w <= 0 || shape_h <= 0) return ml_fail(ML_ERR_ARG, "empty tool shape");
    if (ml_sm_count() <= 0) return ml_fail(ML_ERR_NO_DEVICE, "no CUDA device");
    Arena& A = g_arena;
    std::lock_guard<std::mutex> g(A.mu);
    const long long n = (long long)width * height, nwords = (n + 63) >> 6;
    const size_t es = tri_elem(tri_dtype), ws = ml_raster_workspace_bytes(ntri);
    const size_t b_tri = (size_t)ntri * 6 * es, b_clip = (size_t)ntri * 12 * es;
    const size_t b_depth = (size_t)depth_w * depth_h * sizeof(float), b_shape = (size_t)shape_w * shape_h;
    Trace tr;
    ML_TRY(A.begin(Arena::padded(b_tri) + Arena::padded(b_clip) + Arena::padded(b_depth) + Arena::padded(b_shape) +
                   Arena::padded((size_t)nwords * 64) + 2 * Arena::padded((size_t)nwords * 8) + Arena::padded(ws) + 1024));
    tr.mark("arena");
    void* d_tri = A.take<void>(b_tri);
    void* d_clip = A.take<void>(b_clip);
    float* d_depth = A.take<float>(b_depth);
    uint8_t* d_shape = A.take<uint8_t>(b_shape);
    uint8_t* d_hit = A.take<uint8_t>((size_t)nwords * 64);
    unsigned long long* d_bits = A.take<unsigned long long>((size_t)nwords * 8);
    unsigned long long* d_list = A.take<unsigned long long>((size_t)nwords * 8);
    void* d_ws = A.take<void>(ws);
    unsigned long long* d_ctr = A.take<unsigned long long>(64);
    ML_CUDA(cudaMemsetAsync(d_hit, 0, (size_t)nwords * 64, A.s_run));
    ML_CUDA(cudaMemsetAsync(d_ctr, 0, 64, A.s_run));
    ML_TRY(A.upload(d_depth, depth, b_depth, A.s_up));
    ML_TRY(A.upload(d_shape, shape, b_shape, A.s_up));
    ML_TRY(A.upload(d_clip, tri_clip, b_clip, A.s_up));
    ML_TRY(A.upload(d_tri, tri_xy, b_tri, A.s_up));
    tr.mark("uploads (staged, pipelined)", A.s_up, A.s_run);
    ML_CUDA(cudaEventRecord(A.ev, A.s_up));
    ML_CUDA(cudaStreamWaitEvent(A.s_run, A.ev, 0));
    ml_tea_params tp;
    memset(&tp, 0, sizeof tp);
    tp.ww = ww; tp.wh = wh; tp.eps = eps; tp.sfx = sfx; tp.sfy = sfy; tp.bx = bx; tp.by = by;
    tp.depth = d_depth; tp.shape = d_shape;
    tp.depth_w = depth_w; tp.depth_h = depth_h; tp.shape_w = shape_w; tp.shape_h = shape_h;
    tp.eps_f32 = eps_f32;
    // data = mask = NULL: the kernel records the stroke's texels in the zeroed scratch plane only
    ML_TRY(ml_raster_tea(d_tri, d_clip, tri_dtype, ntri, width, height, 0, height, &tp, nullptr, esize, value_bits,
                         nullptr, d_hit, (uint64_t*)d_ctr, d_ws, ws, A.s_run));
    tr.mark("classify + direct TEA kernel", A.s_run);
    long long newly = 0;
    unsigned long long c[4];                               // [1] = fragments offered (KN:158-161, 203)
    ML_TRY(write_back(A, d_hit, n, d_bits, d_list, d_ctr, c, edited, mask, data, esize, value_bits, &newly));
    tr.mark("pack + download + apply");
    if (edited_count) *edited_count = newly;
    if (fragments) *fragments = (int64_t)c[1];
    return ML_OK;
}

}  // extern "C"
