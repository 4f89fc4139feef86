// tcgen05 (5th-gen tensor core) bf16 gather-GEMM for sm_100a.
//
//   D[r, n] = epi( sum_k A[r,k] * B[n,k] ),  bf16 operands, fp32 accumulation in TMEM.
//
// Structure (one CTA = one 128 x BN output tile, one K split):
//   warps 0-3 : producers — gather the A rows (implicit 3x3 conv with select-on-read,
//               or plain rows) and the B rows (weights) with 16-byte cp.async straight
//               into 128B-swizzled K-major shared memory (the canonical UMMA SW128
//               layout); a stage is published with fence.proxy.async + mbarrier arrive.
//               After the main loop the same warps run the epilogue: tcgen05.ld of
//               their 32 TMEM lanes -> fused epilogue (bias, time bias, cached-stat
//               GN+SiLU, step update, residual) -> global stores.
//   warp 4    : TMEM allocator + MMA issuer (one elected thread issues
//               tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 per instruction;
//               tcgen05.commit frees smem stages and finally signals the epilogue).
// Split-K partials go to a workspace and the last CTA of a tile reduces them in fixed
// split order (bitwise deterministic). The A gather cannot use TMA tiles: rows are
// scattered active pixels whose halo reads select between the fresh compact buffer
// and the step's cache slab per pixel.
#include "fis_tc.cuh"
#include "fis_tma.cuh"

// weight tensor maps (cached per buffer), defined with the persistent GEMM
const CUtensorMap* fis_weight_map(const void* base, long long n, long long k, long long ld, int box);
int fis_tma_a_encode(const fis_gemm_args* a, CUtensorMap* ta, CUtensorMap* ta2);

namespace fis {
namespace tc {

constexpr int PRODUCERS = 256, THREADS = 288, MMA_WARP = 8;

// X3 (fp32 on the tensor cores, 3xTF32): a K block is 32 fp32 (one 128-byte SW128 row, like 64
// bf16); every operand tile exists twice in the stage, as its tf32-rounded "big" part and the fp32
// remainder "small" (the producers split their own rows in place after cp.async lands), and each
// K block issues big*big + big*small + small*big tf32 MMAs into the fp32 accumulator.
template <int BN, bool X3 = false>
struct Smem {
    static constexpr int A_BYTES = BM * 128 * (X3 ? 2 : 1);  // [big][small] when X3
    static constexpr int B_BYTES = BN * 128 * (X3 ? 2 : 1);
    static constexpr int A_PART = BM * 128, B_PART = BN * 128;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = X3 ? 3 : 4;
    static constexpr int EPI = BN * 32;  // per-column epilogue tables
    static constexpr int SEL = BM * 2 * 9 * 4;  // per-row, per-segment, per-tap select-on-read table
    // split-K receive buffer (dedicated: peers push into it while this CTA's main loop may still
    // run): S - 1 row slices of ceil(BM / S) rows x (BN + 4) fp32, maximised over S = 2..16
    static constexpr int rx_bytes(int S) { return (S - 1) * ((BM + S - 1) / S) * (BN + 4) * 4; }
    static constexpr int rx_max(int S) { return S > 16 ? 0 : (rx_bytes(S) > rx_max(S + 1) ? rx_bytes(S) : rx_max(S + 1)); }
    static constexpr int RX = rx_max(2);
    static constexpr int BASE = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/ + EPI + SEL + 16;
    static constexpr int TOTAL = BASE + RX;  // with the split-K receive buffer
};

// Phase timestamps (%globaltimer, ns) of CTA (0,0,0) for profiling the fixed per-launch cost;
// enabled with fis_trace(1), read with fis_trace_read().
__device__ int g_trace_on = 0;
__device__ unsigned long long g_trace[16];
__device__ unsigned long long g_trace_cta[512][4];  // per CTA: entry, mainloop done, cluster sync 1, exit
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifdef FIS_TRACE
__device__ __forceinline__ void trace(int slot) {
    if (g_trace_on && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) g_trace[slot] = gtime();
}
__device__ __forceinline__ void trace_cta(int slot) {
    if (g_trace_on) {
        const int id = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        if (id < 512) g_trace_cta[id][slot] = gtime();
    }
}
#else  // production build: no probes (each is a global load of g_trace_on on thread 0's path)
__device__ __forceinline__ void trace(int) {}
__device__ __forceinline__ void trace_cta(int) {}
#endif

__device__ __forceinline__ void tc_tma2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_tma4d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// amode (A staging): 0 cp.async by the producer threads (gathered / select-on-read rows);
// 1 TMA box {64 x 128} of contiguous rows; 2 dense 3x3 conv, one 4-D box per tap (TMA zero fill =
// the conv padding). With TMA A, thread 0 alone feeds the pipeline (full barrier count 1).
constexpr int AM_CPASYNC = 0, AM_ROWS = 1, AM_CONV = 2;

// tma_b: the B tile {64 x BN} of each stage is one TMA load (thread 0, expect_tx on the stage's
// full barrier) instead of BN rows of cp.async (weights stream faster; fewer producer instructions)
__device__ __forceinline__ float tf32_big(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// split this thread's 16-byte chunk at byte offset off of a raw fp32 tile (in the "small" half):
// big -> off - part_bytes, small stays at off (x - big is exact in fp32)
__device__ __forceinline__ void x3_split(unsigned char* small_tile, int part_bytes, uint32_t off) {
    float4 x = *(float4*)(small_tile + off);
    float4 b = make_float4(tf32_big(x.x), tf32_big(x.y), tf32_big(x.z), tf32_big(x.w));
    *(float4*)(small_tile - part_bytes + off) = b;
    // the remainder rounded to tf32 too (the tensor core would truncate it)
    *(float4*)(small_tile + off) =
        make_float4(tf32_big(x.x - b.x), tf32_big(x.y - b.y), tf32_big(x.z - b.z), tf32_big(x.w - b.w));
}

template <int BN, bool X3>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const fis_gemm_args a, const __grid_constant__ CUtensorMap tmb, int tma_b,
                   const __grid_constant__ CUtensorMap tma0, const __grid_constant__ CUtensorMap tma1, int amode) {
    using SM = Smem<BN, X3>;
    constexpr int ES = X3 ? 4 : 2;             // operand element bytes
    constexpr int BKE = 128 / ES;              // K elements per K block (one 128-byte row)
    constexpr int EPC = 16 / ES;               // K elements per 16-byte chunk
    // X3: the tensor core's fp32 accumulate truncates (~2^-24 per MMA, linear in the K steps), so
    // the big*big products of K block i go to accumulator i % NBIG and both small-product terms to
    // their own accumulator; the epilogue sums them in fp32 (round to nearest), fixed order
    constexpr int NBIG = X3 ? 512 / BN - 1 : 1;
    constexpr int TCOLS = X3 ? 512 : (BN < 32 ? 32 : BN);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(smem + SM::STAGES * SM::STAGE);
    uint64_t* empty = full + SM::STAGES;
    uint64_t* done = empty + SM::STAGES;
    uint64_t* rx_bar = done + 1;  // split-K: peers' partial row slices landed (complete_tx)
    uint32_t* tmem_slot = (uint32_t*)(rx_bar + 1);
    int* last_flag = (int*)(tmem_slot + 1);  // followed by the epilogue tables

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ int s_ltr;
    if (tid == 0) { trace(0); trace_cta(0); s_ltr = ltr_begin(1); }
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const int kblocks = (a.k + BKE - 1) / BKE;
    const int kper = (kblocks + a.splits - 1) / a.splits;
    const int kb0 = blockIdx.z * kper, kb1 = min(kblocks, kb0 + kper);
    const int nk = max(0, kb1 - kb0);

    if (tid == 0) {
        for (int s = 0; s < SM::STAGES; s++) {
            mbar_init(full + s, amode ? 1 : PRODUCERS + (tma_b ? 1 : 0));
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        mbar_init(rx_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) trace(1);
    // split-K: announce this CTA's barriers initialised; the matching wait comes right before the
    // first push into a peer (long satisfied by then)
    if (a.splits > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    // gather metadata of the producer's row: pixel + (CONV) the select-on-read decision of every
    // tap of both concat segments, in a shared table; read before the programmatic-launch wait
    // when the row/index lists are static (they are inside a captured edit step)
    int* seltab = (int*)(((uintptr_t)(smem + SM::STAGES * SM::STAGE + 256 + SM::EPI) + 15) & ~(uintptr_t)15);
    const int ar = tid >> 1, half_id = tid & 1;
    int row_p = 0;
    bool row_valid = false;
    auto build_meta = [&]() {
        if (warp >= MMA_WARP) return;
        const int r = m0 + ar;
        row_valid = r < a.m;
        row_p = row_valid ? (a.rows ? __ldg(a.rows + r) : r) : 0;
        if (a.a_mode == FIS_A_CONV3X3 && half_id < a.nsrc) build_sel(a, row_p, half_id, seltab + (ar * 2 + half_id) * 9);
    };
    if (a.static_meta) build_meta();
    // the step counter is written by the host before the step (outside the captured graph), so it
    // is read before the wait: its load latency overlaps the previous kernel too
    const int t = cur_step(a.step);
    const int ls = s_ltr;
    if (tid == 0) ltr(ls, 1);
    // weights (no kernel writes them): the first stages' B tiles go straight into shared memory and
    // the rest into L2 while the previous kernel still runs; with TMA A the stage's A bytes are
    // expected here too (issued after the wait)
    const int pre = tma_b ? min(nk, SM::STAGES) : 0;
    if (tid == 0)
        for (int i = 0; i < pre; i++) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + i)),
                         "r"((uint32_t)(BN * 128 + (amode ? SM::A_BYTES : 0)))
                         : "memory");
            tc_tma2d(smem_u32(smem) + i * SM::STAGE + SM::A_BYTES, &tmb, (kb0 + i) * BKE, n0, full + i);
        }
    if (tma_b && warp == MMA_WARP + 0 && lane == 0 && !a.b.step_stride) {
        for (int i = pre; i < nk; i++) tma_prefetch2d(&tmb, (kb0 + i) * BKE, n0);
    }
    pdl_trigger();
    pdl_wait();  // everything above (barrier init, TMEM alloc, static metadata) overlaps the previous kernel
    if (tid == 0) ltr(ls, 2);
    if (!a.static_meta) build_meta();
    if (tid == 0) trace(2);

    if (warp < MMA_WARP && amode) {
        // ------------------------------------------------------------ TMA A (+ B) producer: thread 0
        if (tid == 0) {
            const uint32_t sbase = smem_u32(smem);
            const int cin0 = a.nsrc > 0 ? a.src[0].c : 0, cin = cin0 + (a.nsrc > 1 ? a.src[1].c : 0);
            const int ow = a.out_w, ohw = a.out_h * a.out_w;
            const int img = amode == AM_CONV ? m0 / ohw : 0;
            const int y0 = amode == AM_CONV && ohw >= BM ? (m0 - img * ohw) / ow : 0;
            for (int i = 0; i < nk; i++) {
                const int s = i % SM::STAGES;
                const int k0 = (kb0 + i) * BKE;
                const uint32_t sa = sbase + s * SM::STAGE;
                if (i >= SM::STAGES) {
                    mbar_wait(empty + s, ((i / SM::STAGES) & 1) ^ 1);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)),
                                 "r"((uint32_t)(BN * 128 + SM::A_BYTES))
                                 : "memory");
                    tc_tma2d(sa + SM::A_BYTES, &tmb, k0, n0, full + s);
                }
                if (amode == AM_ROWS) {
                    tc_tma2d(sa, &tma0, k0, m0, full + s);
                } else {
                    const int tap = k0 / cin;
                    int c = k0 - tap * cin;
                    const bool seg1 = c >= cin0;
                    c -= seg1 ? cin0 : 0;
                    tc_tma4d(sa, seg1 ? &tma1 : &tma0, c, tap % 3 - 1, y0 + tap / 3 - 1, img, full + s);
                }
                if (i == 0) trace(3);
            }
        }
    } else if (warp < MMA_WARP) {
        // ------------------------------------------------------------ producers
        const char* abase = a.a.ptr ? ref_base(a.a, t) : nullptr;
        const char* f0 = a.nsrc > 0 && a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
        const char* c0p = a.nsrc > 0 && a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
        const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
        const char* c1p = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
        const char* bbase = ref_base(a.b, t);
        const int cin = a.a_mode == FIS_A_CONV3X3 ? a.src[0].c + (a.nsrc > 1 ? a.src[1].c : 0) : a.k;
        const uint32_t sbase = smem_u32(smem);
        // thread -> (row, half): two threads share a 128-byte row, 4 chunks of 16 B each
        const int j0 = half_id * 4;
        __syncwarp();  // the two threads of a row each built one segment's table entries
        const int* mysel = seltab + ar * 2 * 9;
        const int src0c = a.nsrc > 0 ? a.src[0].c : 0;
        const int bn = n0 + ar;
        const char* brow = bbase + (long long)bn * a.b.ld * ES;
        constexpr int LAG = 2;  // X3: stages of this thread's copies in flight before it splits one
        auto x3_publish = [&](int q) {  // split this thread's chunks of stage q in place, publish it
            unsigned char* st = smem + (q % SM::STAGES) * SM::STAGE;
#pragma unroll
            for (int j = j0; j < j0 + 4; j++) {
                x3_split(st + SM::A_PART, SM::A_PART, sw128_off(ar, j));
                if (ar < BN) x3_split(st + SM::A_BYTES + SM::B_PART, SM::B_PART, sw128_off(ar, j));
            }
            fence_async_smem();
            mbar_arrive(full + q % SM::STAGES);
        };
        for (int i = 0; i < nk; i++) {
            const int s = i % SM::STAGES;
            const int k0 = (kb0 + i) * BKE;
            if (i >= SM::STAGES) mbar_wait(empty + s, ((i / SM::STAGES) & 1) ^ 1);
            // X3: raw fp32 rows land in the "small" halves and are split in place
            const uint32_t sa = sbase + s * SM::STAGE + (X3 ? SM::A_PART : 0);
            const uint32_t sb = sbase + s * SM::STAGE + SM::A_BYTES + (X3 ? SM::B_PART : 0);
            const char* src = nullptr;
            if (row_valid) {
                if (a.a_mode == FIS_A_ROWS) {
                    if (k0 < a.k) src = abase + ((long long)row_p * a.a.ld + k0) * ES;
                } else {
                    const int tap = k0 / cin;
                    int c = k0 - tap * cin;
                    const int seg = c >= src0c ? 1 : 0;
                    c -= seg ? src0c : 0;
                    const int sel = mysel[seg * 9 + tap];
                    if (sel != SEL_ZERO) {
                        const fis_src& sr = a.src[seg];
                        if (sel >= 0) src = (seg ? f1 : f0) + ((long long)sel * sr.fresh.ld + c) * ES;
                        else src = (seg ? c1p : c0p) + ((long long)(-2 - sel) * sr.cache.ld + c) * ES;
                    }
                }
            }
#pragma unroll
            for (int j = j0; j < j0 + 4; j++) {
                const bool ok = src != nullptr && (a.a_mode == FIS_A_CONV3X3 || k0 + j * EPC < a.k);
                cp_async16(sa + sw128_off(ar, j), ok ? (const void*)(src + j * 16) : (const void*)bbase, ok);
            }
            if (tma_b) {
                if (tid == 0 && i >= SM::STAGES) {  // the first stages' B tiles were issued before the wait
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)),
                                 "r"((uint32_t)(BN * 128))
                                 : "memory");
                    tc_tma2d(sb, &tmb, k0, n0, full + s);
                }
            } else if (ar < BN) {  // B: weight row ar of this N tile
#pragma unroll
                for (int j = j0; j < j0 + 4; j++) {
                    const bool ok = bn < a.n && k0 + j * EPC < a.k;
                    cp_async16(sb + sw128_off(ar, j), ok ? (const void*)(brow + (long long)(k0 + j * EPC) * ES)
                                                         : (const void*)bbase,
                               ok);
                }
            }
            if (X3) {
                cp_commit();
                if (i >= LAG) {
                    cp_wait<LAG>();
                    x3_publish(i - LAG);
                }
            } else {
                // the barrier counts this thread's arrival when all its prior cp.async have landed:
                // no thread-side wait, SM::STAGES stages of loads stay in flight
                cp_async_arrive_noinc(full + s);
            }
            if (tid == 0 && i == 0) trace(3);
        }
        if (X3) {  // drain: split and publish the last LAG stages
            cp_wait<0>();
            for (int q = nk - LAG < 0 ? 0 : nk - LAG; q < nk; q++) x3_publish(q);
        }
    } else {
        // ------------------------------------------------------------ MMA issuer
        // c = F32; a, b = BF16 (1) or TF32 (2); K-major; N >> 3; M >> 4
        const uint32_t fmt = X3 ? 2u : 1u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);
        const uint32_t sbase = smem_u32(smem);
        for (int i = 0; i < nk; i++) {
            const int s = i % SM::STAGES;
            mbar_wait(full + s, (i / SM::STAGES) & 1);
            if (lane == 0 && i == 0) { trace(4); ltr(ls, 3); }
            if (lane == 0 && i == nk - 1) { trace(5); ltr(ls, 4); }
            tc_fence_after();
            if (lane == 0) {
                const uint32_t sa = sbase + s * SM::STAGE;
                const uint32_t sb = sa + SM::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {  // 4 MMAs of 32 bytes of K (16 bf16 / 8 tf32)
                    const uint64_t ad = sw128_desc(sa + kk * 32), bd = sw128_desc(sb + kk * 32);
                    const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                    if (X3) {
                        const uint64_t as = sw128_desc(sa + SM::A_PART + kk * 32);
                        const uint64_t bs = sw128_desc(sb + SM::B_PART + kk * 32);
                        const uint32_t dbig = tmem + (uint32_t)((i % NBIG) * BN), dsmall = tmem + (uint32_t)(NBIG * BN);
                        const uint32_t acc_big = (i >= NBIG || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p, q, r;\nsetp.ne.b32 p, %7, 0;\nsetp.eq.b32 q, 0, 0;\nsetp.ne.b32 r, %8, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%1], %2, %4, %6, p;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %5, %6, q;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %3, %4, %6, r;\n}\n" ::"r"(dbig),
                            "r"(dsmall), "l"(as), "l"(ad), "l"(bd), "l"(bs), "r"(idesc), "r"(acc), "r"(acc_big));
                    } else {
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(empty + s))
                             : "memory");
            }
            __syncwarp();
        }
        if (lane == 0) {
            if (nk > 0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(done))
                             : "memory");
            else
                mbar_arrive(done);
        }
        __syncwarp();
    }

    // ---------------------------------------------------------------- epilogue
    EpiTab tb;
    {
        unsigned char* ep = (unsigned char*)(last_flag + 4);
        ep = (unsigned char*)(((uintptr_t)ep + 15) & ~(uintptr_t)15);
        tb.mean = (float*)ep;
        tb.rstd = tb.mean + BN;
        tb.bias = (float*)(tb.rstd + BN);
        tb.b2 = tb.bias + BN;
        tb.gamma = tb.b2 + BN;
        tb.beta = tb.gamma + BN;
    }
    const EpiCtx e = make_epi(a, t);
    const int S = a.splits > 1 ? a.splits : 1;  // split-K CTAs of this tile = one cluster along z
    // fp32 partial tile [BM][BN+4] staged in the (now idle) pipeline buffers
    constexpr int PLD = BN + 4;
    float* part = (float*)smem;
    if (warp < MMA_WARP) {
        // stage per-column parameters while the MMAs drain
        for (int c = tid; c < BN; c += PRODUCERS) {
            const int n = n0 + c;
            const bool ok = n < a.n;
            tb.bias[c] = ok && a.bias ? __ldg(a.bias + n) : 0.f;
            tb.b2[c] = ok && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n) : 0.f;
            if (a.epi == FIS_EPI_GN_SILU && ok) {
                const int g = n / e.cpg;
                // cached-stat GN folded into one fma per element: y = v * scale + shift
                const float rstd = (float)(1.0 / sqrt((double)e.var[g] + (double)a.eps));
                const float scale = rstd * __ldg(a.gamma + n);
                tb.mean[c] = scale;
                tb.rstd[c] = fmaf(-e.mean[g], scale, __ldg(a.beta + n));
                tb.gamma[c] = 0.f;
                tb.beta[c] = 0.f;
            } else {
                tb.mean[c] = 0.f; tb.rstd[c] = 0.f; tb.gamma[c] = 0.f; tb.beta[c] = 0.f;
            }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (tid == 0) trace(10);
        mbar_wait(done, 0);
        if (tid == 0) { trace(6); trace_cta(1); ltr(ls, 5); }
        tc_fence_after();
        const int quarter = warp & 3, half = warp >> 2;
        const int lr = quarter * 32 + lane;
        // all TMEM loads of this thread's row segment first, one wait (latency paid once)
        constexpr int HC = BN / 2;  // columns per warp half
        uint32_t u[HC];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + half * HC;
        if (X3 && nk > 0) {  // small-product accumulator + the big*big accumulators in use, in order
            float accv[HC];
            const int nb = nk < NBIG ? nk : NBIG;
            for (int b = -1; b < nb; b++) {
                const uint32_t ta = taddr + (uint32_t)((b < 0 ? NBIG : b) * BN);
#pragma unroll
                for (int q = 0; q < HC / 16; q++) {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(u[16 * q + 0]), "=r"(u[16 * q + 1]), "=r"(u[16 * q + 2]), "=r"(u[16 * q + 3]),
                          "=r"(u[16 * q + 4]), "=r"(u[16 * q + 5]), "=r"(u[16 * q + 6]), "=r"(u[16 * q + 7]),
                          "=r"(u[16 * q + 8]), "=r"(u[16 * q + 9]), "=r"(u[16 * q + 10]), "=r"(u[16 * q + 11]),
                          "=r"(u[16 * q + 12]), "=r"(u[16 * q + 13]), "=r"(u[16 * q + 14]), "=r"(u[16 * q + 15])
                        : "r"(ta + 16 * q));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < HC; j++) accv[j] = b < 0 ? __uint_as_float(u[j]) : __fadd_rn(accv[j], __uint_as_float(u[j]));
            }
#pragma unroll
            for (int j = 0; j < HC; j++) u[j] = __float_as_uint(accv[j]);
        } else {
#pragma unroll
        for (int q = 0; q < HC / 16; q++) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(u[16 * q + 0]), "=r"(u[16 * q + 1]), "=r"(u[16 * q + 2]), "=r"(u[16 * q + 3]),
                  "=r"(u[16 * q + 4]), "=r"(u[16 * q + 5]), "=r"(u[16 * q + 6]), "=r"(u[16 * q + 7]),
                  "=r"(u[16 * q + 8]), "=r"(u[16 * q + 9]), "=r"(u[16 * q + 10]), "=r"(u[16 * q + 11]),
                  "=r"(u[16 * q + 12]), "=r"(u[16 * q + 13]), "=r"(u[16 * q + 14]), "=r"(u[16 * q + 15])
                : "r"(taddr + 16 * q));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        {
            // stage the fp32 tile (the split-K partial, or the whole tile when S == 1) in the idle
            // pipeline buffers; the stores below run columns-fastest across threads (coalesced), not
            // one row per thread (a warp's 32 row stores are 32 separate lines: ~4.5 us per tile)
            float* p = part + lr * PLD + half * HC;
#pragma unroll
            for (int q = 0; q < HC / 4; q++)
                *(float4*)(p + 4 * q) = nk > 0 ? make_float4(__uint_as_float(u[4 * q]), __uint_as_float(u[4 * q + 1]),
                                                             __uint_as_float(u[4 * q + 2]), __uint_as_float(u[4 * q + 3]))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    if (tid == 0) { trace(8); ltr(ls, 6); }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) { trace(9); ltr(ls, 8); }
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
    if (tid == 0) ltr(ls, 9);
    // fused epilogue of tile rows [rbeg, rend) from an fp32 staging buffer (row lr at src + (lr - rbeg) * PLD),
    // 16-column chunks; transposed outputs (V^T of a fused QKV, or d_trans) go rows-fastest across threads so a
    // warp stores 32 consecutive rows of each column, row-major outputs columns-fastest
    const bool tile_trans = a.d_trans || (a.d2_trans && a.n_split > 0 && n0 >= a.n_split);
    // plain bf16 row-major output with bias only (projections, most convs): a compact inline path
    const bool plain = a.epi == FIS_EPI_NONE && a.alpha == 1.0f && !e.pre && !e.res && !e.bias2 && !a.d_rows &&
                       !tile_trans && a.n_split == 0 && a.d.dtype == FIS_BF16 && (a.d.ld % 8) == 0 &&
                       (((uintptr_t)e.d) & 15) == 0 && (a.n % 16) == 0;
    auto epi_rows = [&](const float* src, int rbeg, int rend) {
        const int chunks = BN / 16;
        const int nrows = rend - rbeg;
        if (plain) {
#pragma unroll 1
            for (int item = tid; item < nrows * chunks; item += THREADS) {
                const int lr = rbeg + item / chunks, cb = (item % chunks) * 16;
                const int r = m0 + lr;
                if (r >= a.m || n0 + cb >= a.n) continue;
                const float* q = src + (lr - rbeg) * PLD + cb;
                uint4 o[2];
                __nv_bfloat162* h = (__nv_bfloat162*)o;
#pragma unroll
                for (int k4 = 0; k4 < 4; k4++) {
                    const float4 f = *(const float4*)(q + 4 * k4);
                    h[2 * k4] = __floats2bfloat162_rn(__fadd_rn(f.x, tb.bias[cb + 4 * k4]),
                                                      __fadd_rn(f.y, tb.bias[cb + 4 * k4 + 1]));
                    h[2 * k4 + 1] = __floats2bfloat162_rn(__fadd_rn(f.z, tb.bias[cb + 4 * k4 + 2]),
                                                          __fadd_rn(f.w, tb.bias[cb + 4 * k4 + 3]));
                }
                uint4* dst = (uint4*)((__nv_bfloat16*)e.d + (long long)r * a.d.ld + n0 + cb);
                dst[0] = o[0];
                dst[1] = o[1];
            }
            return;
        }
        for (int item = tid; item < nrows * chunks; item += THREADS) {
            const int lr = rbeg + (tile_trans ? item % nrows : item / chunks);
            const int cb = (tile_trans ? item / nrows : item % chunks) * 16;
            const int r = m0 + lr;
            if (r >= a.m || n0 + cb >= a.n) continue;
            float v[16];
            const float* q = src + (lr - rbeg) * PLD + cb;
#pragma unroll
            for (int k4 = 0; k4 < 4; k4++) {
                const float4 f = *(const float4*)(q + 4 * k4);
                v[4 * k4] = f.x; v[4 * k4 + 1] = f.y; v[4 * k4 + 2] = f.z; v[4 * k4 + 3] = f.w;
            }
            row_epilogue_any(a, e, tb, r, cb, n0, v);
        }
    };
    if (S == 1) {
        epi_rows(part, 0, min(BM, a.m - m0));
    } else {
        // split-K over the S CTAs of a cluster, deterministic: CTA z owns rows [z*rows_per, ...) of
        // the tile; every CTA pushes each peer's row slice of its fp32 partial into that peer's
        // dedicated receive buffer with one DSMEM bulk copy (complete_tx on the peer's rx_bar), so
        // no cluster-wide barrier sits between the partials and the reduction; the owner sums the S
        // partials in split order (bitwise the same as a sequential reduction) and runs the epilogue
        uint32_t rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        // only the tile's valid rows are exchanged (M = 64 / 100-row GEMMs at batch 1 would push
        // 50% / 22% padding rows through the ~20 B/cycle DSMEM port)
        const int vrows = min(BM, a.m - m0);
        const int rows_per = (vrows + S - 1) / S;
        const int rbeg = min(vrows, (int)rank * rows_per), rend = min(vrows, rbeg + rows_per);
        float* rx = (float*)(((uintptr_t)(seltab + BM * 2 * 9) + 15) & ~(uintptr_t)15);
        const uint32_t slice_floats = (uint32_t)rows_per * PLD;
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' rx_bar initialised
        if (tid == 0) {
            // incoming bytes: S - 1 slices of this CTA's rows
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rx_bar)),
                         "r"((uint32_t)((S - 1) * (rend - rbeg) * PLD * 4))
                         : "memory");
            fence_async_smem();  // generic-proxy partial writes -> bulk-copy reads
            const uint32_t part_s = smem_u32(part), rx_s = smem_u32(rx), bar_s = smem_u32(rx_bar);
            for (int p = 0; p < S; p++) {
                if (p == (int)rank) continue;
                const int pb = min(vrows, p * rows_per), pe = min(vrows, pb + rows_per);
                if (pe <= pb) continue;
                const int slot = (int)rank < p ? (int)rank : (int)rank - 1;  // my slot in peer p's buffer
                uint32_t dst, bar;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(rx_s + slot * slice_floats * 4), "r"(p));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(bar_s), "r"(p));
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "r"(part_s + (uint32_t)(pb * PLD * 4)), "r"((uint32_t)((pe - pb) * PLD * 4)), "r"(bar)
                    : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (rend > rbeg) {
            mbar_wait(rx_bar, 0);
            const int chunks = BN / 16, nrows = rend - rbeg;
            for (int item = tid; item < nrows * chunks; item += THREADS) {
                const int lr = rbeg + (tile_trans ? item % nrows : item / chunks);
                const int cb = (tile_trans ? item / nrows : item % chunks) * 16;
                const int r = m0 + lr;
                if (r >= a.m || n0 + cb >= a.n) continue;
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; j++) v[j] = 0.f;
                for (int z = 0; z < S; z++) {  // split order
                    const float* q = z == (int)rank ? part + lr * PLD + cb
                                                    : rx + (z < (int)rank ? z : z - 1) * slice_floats + (lr - rbeg) * PLD + cb;
#pragma unroll
                    for (int k4 = 0; k4 < 4; k4++) {
                        const float4 f = *(const float4*)(q + 4 * k4);
                        v[4 * k4] += f.x; v[4 * k4 + 1] += f.y; v[4 * k4 + 2] += f.z; v[4 * k4 + 3] += f.w;
                    }
                }
                row_epilogue_any(a, e, tb, r, cb, n0, v);
            }
        }
        // this CTA's outgoing copies must have read its partial before the shared memory goes away
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (tid == 0) { trace(7); trace_cta(3); ltr(ls, 7); }
}

template <int BN, bool X3>
int launch(const fis_gemm_args* a, cudaStream_t stream) {
    using SM = Smem<BN, X3>;
    const int smem = a->splits > 1 ? SM::TOTAL : SM::BASE;
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(gemm_tc_kernel<BN, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL) !=
            cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        cudaFuncSetAttribute(gemm_tc_kernel<BN, X3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        configured = true;
    }
    const int S = a->splits > 1 ? a->splits : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a->n + BN - 1) / BN, (a->m + BM - 1) / BM, S);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (S > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = S;
        na++;
    }
    if (fis_pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    static int tma_off = getenv("FIS_TC_TMA_B") && getenv("FIS_TC_TMA_B")[0] == '0';
    const CUtensorMap* tm = nullptr;
    if (!tma_off && a->b.dtype == FIS_BF16 && !a->b.step_stride && (a->b.ld % 8) == 0)
        tm = fis_weight_map(a->b.ptr, a->n, a->k, a->b.ld, BN);
    CUtensorMap none, ta, ta2;
    std::memset(&none, 0, sizeof(none));
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&ta2, 0, sizeof(ta2));
    static int tma_a_off = getenv("FIS_TC_TMA_A") && getenv("FIS_TC_TMA_A")[0] == '0';
    const int amode = (!X3 && tm && !tma_a_off) ? fis_tma_a_encode(a, &ta, &ta2) : AM_CPASYNC;
    return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, X3>, *a, tm ? *tm : none, tm ? 1 : 0, ta, ta2, amode) ==
                   cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}

// How many clusters of S CTAs (split-K) the device co-schedules for this kernel, S = 1..16
// (GPC packing: ~18 SMs per GPC, 1 CTA per SM). Cached per BN.
template <int BN, bool X3>
int active_clusters(int S) {
    using SM = Smem<BN, X3>;
    static int table[17] = {0};
    if (S < 1 || S > 16) return 0;
    if (table[S]) return table[S];
    cudaFuncSetAttribute(gemm_tc_kernel<BN, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::TOTAL);
    cudaFuncSetAttribute(gemm_tc_kernel<BN, X3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, S);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SM::TOTAL;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 1;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = S;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<BN, X3>, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    table[S] = n > 0 ? n : -1;
    return table[S];
}

// Largest S such that all tiles' clusters run in one wave and each split keeps >= 3 K blocks.
template <int BN, bool X3>
int choose_splits(long long tiles, long long kb) {
    int best = 1;
    for (int S = 2; S <= 16; S++) {
        if (kb / S < 3) break;
        const int ac = active_clusters<BN, X3>(S);
        if (ac >= tiles) best = S;
    }
    return best;
}


}  // namespace tc
}  // namespace fis

// TC path requirements: bf16 A sources and B; 16-byte aligned rows; CONV segments
// whose channel counts are multiples of 64 (a 64-wide K block never straddles a tap
// or a concat boundary); ROWS mode any K (zero-filled tail).
int fis_gemm_tc_supported(const fis_gemm_args* a) {
    if (a->b.dtype != FIS_BF16 || (a->b.ld % 8)) return 0;
    if (a->n_split > 0 && (a->n_split % 32)) return 0;
    if (a->a_mode == FIS_A_ROWS) {
        if (a->a.dtype != FIS_BF16 || (a->a.ld % 8)) return 0;
        return 1;
    }
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.c % 64) return 0;
        if (s.fresh.dtype != FIS_BF16 || (s.fresh.ld % 8)) return 0;
        if (s.index && (s.cache.dtype != FIS_BF16 || (s.cache.ld % 8))) return 0;
    }
    return 1;
}

int fis_gemm_tc_choose_splits(int m, int n, int k) {
    const long long kb = (k + fis::tc::BK - 1) / fis::tc::BK;
    if (n <= 64) return fis::tc::choose_splits<64, false>((long long)((m + 127) / 128) * ((n + 63) / 64), kb);
    return fis::tc::choose_splits<128, false>((long long)((m + 127) / 128) * ((n + 127) / 128), kb);
}

int fis_gemm_tc_launch(const fis_gemm_args* a, cudaStream_t stream) {
    if (!fis_gemm_tc_supported(a)) return FIS_ERR_UNSUPPORTED;
    if (a->n <= 64) return fis::tc::launch<64, false>(a, stream);
    return fis::tc::launch<128, false>(a, stream);
}

// 3xTF32 path (fp32 operands on the tensor cores): fp32 A sources and B with 16-byte aligned rows;
// CONV segments whose channel counts are multiples of 32 (a 32-wide fp32 K block never straddles a
// tap or a concat boundary); ROWS mode any K. 128 x 64 tiles.
int fis_gemm_tf32_supported(const fis_gemm_args* a) {
    if (a->b.dtype != FIS_F32 || (a->b.ld % 4)) return 0;
    if (a->n_split > 0 && (a->n_split % 32)) return 0;
    if (a->a_mode == FIS_A_ROWS) return a->a.dtype == FIS_F32 && (a->a.ld % 4) == 0;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.c % 32) return 0;
        if (s.fresh.dtype != FIS_F32 || (s.fresh.ld % 4)) return 0;
        if (s.index && (s.cache.dtype != FIS_F32 || (s.cache.ld % 4))) return 0;
    }
    return 1;
}

int fis_gemm_tf32_choose_splits(int m, int n, int k) {
    const long long kb = (k + 31) / 32;
    return fis::tc::choose_splits<64, true>((long long)((m + 127) / 128) * ((n + 63) / 64), kb);
}

int fis_gemm_tf32_launch(const fis_gemm_args* a, cudaStream_t stream) {
    if (!fis_gemm_tf32_supported(a)) return FIS_ERR_UNSUPPORTED;
    return fis::tc::launch<64, true>(a, stream);
}

FIS_LTR_SETTER(fis_ltr_set_tc)

extern "C" int fis_trace(int on) {
    return cudaMemcpyToSymbol(fis::tc::g_trace_on, &on, sizeof(int)) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}
extern "C" int fis_trace_read_ctas(unsigned long long* out2048) {
    return cudaMemcpyFromSymbol(out2048, fis::tc::g_trace_cta, 512 * 4 * sizeof(unsigned long long)) == cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}
extern "C" int fis_trace_read(unsigned long long* out16) {
    return cudaMemcpyFromSymbol(out16, fis::tc::g_trace, 16 * sizeof(unsigned long long)) == cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}
