// Bulk asynchronous copies (TMA, 1-D form) + mbarrier ring for the whole-atlas streaming kernels.
//
// A read stream whose bytes are consumed once (an outline plane, the owner-id map, an attribute
// plane) does not need registers as its landing zone: ONE elected lane per block keeps STAGES
// `cp.async.bulk.shared::cluster.global` copies of CHUNK bytes in flight into a shared-memory ring
// (SASS: UBLKCP), each completing on the stage's "full" mbarrier; consumer warps wait on the
// barrier's phase parity, read the stage with conflict-free 128-bit LDS, and release it by
// arriving on the stage's "empty" barrier.  Bytes in flight per SM = blocks/SM x STAGES x CHUNK,
// independent of the register budget and of the number of resident warps, which is what the
// register-streaming forms of these kernels ran out of (64 B per thread in flight at 1024
// threads/SM = 64 KB/SM; the id stream of the TEA kernel sat at 0.75 of the HBM peak with it).
//
// Canonical producer / consumer protocol (blackwell guide, "mbarrier producer/consumer pipeline"):
//   stage s of round k (k-th use of the stage): full[s] completes phase k when the copy's bytes
//   have landed; empty[s] completes phase k when all CONSUMER_WARPS have released the stage.
//   Producer before refilling stage s for round k >= 1 waits empty[s] parity (k-1)&1.
//   Consumers of round k wait full[s] parity k&1; before releasing a stage they issue
//   fence.proxy.async (their generic-proxy reads must be ordered before the async-proxy refill).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef ML_DEV
#define ML_DEV __device__ __forceinline__
#endif

ML_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

ML_DEV void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(bar)), "r"(count) : "memory");
}
// make the barrier initialisation visible to the async (TMA) proxy
ML_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
ML_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_addr(bar)) : "memory");
}
ML_DEV void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(bar)), "r"(bytes) : "memory");
}
ML_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n"     /* suspend-time hint: the wait sleeps in hardware */
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" :: "r"(smem_addr(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16; both addresses 16-byte aligned) that
// completes `bytes` of transaction count on `bar`.  Streamed-once data: L2 evict_first policy.
ML_DEV void bulk_g2s(void* dst_smem, const void* src_gmem, unsigned bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_addr(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(policy) : "memory");
}
ML_DEV uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// shared -> global bulk store (bulk async-group completion); the source bytes must have been made
// visible to the async proxy with fence_proxy_async() after the generic-proxy writes
ML_DEV void bulk_s2g(void* dst_gmem, const void* src_smem, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst_gmem), "r"(smem_addr(src_smem)), "r"(bytes) : "memory");
}
ML_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> ML_DEV void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
template <int N> ML_DEV void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory"); }
ML_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Ring bookkeeping shared by producer and consumers: chunk j of this block (j = 0, 1, ...) lives in
// stage j % STAGES during round j / STAGES.
template <int STAGES>
struct RingPos {
    int stage = 0;
    unsigned round = 0;
    ML_DEV void next() { if (++stage == STAGES) { stage = 0; ++round; } }
    ML_DEV unsigned full_parity() const { return round & 1u; }
    ML_DEV unsigned empty_parity() const { return (round + 1u) & 1u; }      // parity of round-1's completion
};

// Block-level ring: `STAGES` buffers of `CHUNK` bytes + barriers.  Lives in (dynamic) shared memory;
// buffers first so that they keep the 128-byte alignment of the allocation.
template <int STAGES, int CHUNK>
struct BulkRing {
    alignas(128) uint8_t buf[STAGES][CHUNK];
    alignas(8) uint64_t full[STAGES];
    alignas(8) uint64_t empty[STAGES];

    // one thread: barriers ready before anybody touches them (follow with __syncthreads())
    ML_DEV void init(unsigned consumer_warps) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1u); mbar_init(&empty[s], consumer_warps); }
        mbar_fence_init();
    }
    // PRODUCER lane: fetch `bytes` from `src` into the ring position `pos` (waits for the stage to be free)
    ML_DEV void produce(const RingPos<STAGES>& pos, const void* src, unsigned bytes, uint64_t policy) {
        if (pos.round > 0) mbar_wait(&empty[pos.stage], pos.empty_parity());
        mbar_arrive_expect_tx(&full[pos.stage], bytes);
        bulk_g2s(buf[pos.stage], src, bytes, &full[pos.stage], policy);
    }
    // PRODUCER lane, several sources per stage (e.g. one slice of each of G planes): arm the stage for
    // `total` bytes, then issue the pieces with fill()
    ML_DEV void begin_fill(const RingPos<STAGES>& pos, unsigned total) {
        if (pos.round > 0) mbar_wait(&empty[pos.stage], pos.empty_parity());
        mbar_arrive_expect_tx(&full[pos.stage], total);
    }
    ML_DEV void fill(const RingPos<STAGES>& pos, unsigned offset, const void* src, unsigned bytes, uint64_t policy) {
        bulk_g2s(buf[pos.stage] + offset, src, bytes, &full[pos.stage], policy);
    }
    // CONSUMER threads: wait until the stage holds its chunk
    ML_DEV const uint8_t* acquire(const RingPos<STAGES>& pos) {
        mbar_wait(&full[pos.stage], pos.full_parity());
        return buf[pos.stage];
    }
    // CONSUMER warps (all lanes call; lane 0 arrives once the warp's reads are done)
    // The stage's next user is the ASYNC proxy (the producer's next cp.async.bulk overwrites it), the reads
    // just done were generic-proxy LDS: a write-after-read across proxies is ordered only by a proxy fence.
    // Measured without it (area_bulk_kernel<1>, 4 KB stages, 16.8 M texels): tens of texels per launch read
    // from the NEXT round's bytes -- mbarrier release semantics alone do not cover the async proxy.
    ML_DEV void release(const RingPos<STAGES>& pos) {
        fence_proxy_async();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[pos.stage]);
    }
};
