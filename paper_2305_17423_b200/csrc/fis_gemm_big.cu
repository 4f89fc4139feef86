// Persistent warp-specialised tcgen05 gather-GEMM for large M (stacked / batched requests).
//
//   D[r, n] = epi( sum_k A[r,k] * B[n,k] ),  bf16 operands, fp32 accumulation in TMEM.
//
// The per-op kernel (fis_gemm_tc.cu) runs one 128 x 128 tile per CTA with split-K clusters:
// right for the batch-1 step (M = 100-400 rows, weight-streaming bound), but at M in the
// thousands (R requests stepped as one batch) it pays a fresh prologue per tile, 1 CTA per SM
// in waves, and 64 flop per L2 byte. This kernel keeps one CTA per SM for the whole GEMM:
//
//   warps 0-3 : A producers. Thread = tile row: per tile it builds the row's select-on-read
//               decisions (3x3 conv taps over the fresh compact rows / the cached slab, image
//               aware), then per 64-wide K block gathers its 128-byte row with cp.async into
//               the SW128 K-major stage (arrival counted on the stage's full barrier).
//   warp 4    : B producer: one thread issues a TMA tile load {64 x BN} of the weights per
//               stage (128-byte swizzle, zero fill past N / K), expect_tx on the full barrier.
//   warp 5    : TMEM allocator + MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN,
//               K=16; commit frees the stage; a tile's last commit signals the epilogue).
//   warps 6-9 : epilogue: tcgen05.ld of the tile's accumulator (TMEM lanes = rows), fused
//               row epilogue (bias, time bias, cached-stat GN + SiLU, step update, residual,
//               QKV split / transposed V) and stores.
// Two TMEM accumulators (2 x BN <= 512 columns) let the epilogue of tile i overlap the main
// loop of tile i+1. Tiles run N-fastest so consecutive CTAs share the gathered A rows in L2.
// BN is a multiple of 16 in [128, 256] dividing N where possible (UMMA N; 320 -> 160,
// 960 -> 240, 1280 -> 256), so no tile column is wasted.
#include "fis_tc.cuh"
#include "fis_tma.cuh"
#include <cstdio>

namespace fis {
namespace big {

using namespace fis::tc;

constexpr int THREADS = 320;
constexpr int A_WARPS = 4, B_WARP = 4, MMA_WARP = 5, EPI_WARP0 = 6;
constexpr int A_BYTES = BM * BK * 2;     // 16 KB
constexpr int SMEM_BUDGET = 200 * 1024;  // pipeline stages
constexpr int MAX_STAGES = 8;
constexpr int ACC_STRIDE = 256;          // TMEM column offset of accumulator 1
constexpr int A_CPASYNC = 0, A_TMA_ROWS = 1, A_TMA_CONV = 2, A_TMA_GATHER = 3;  // how A tiles are staged

// TMA gather4 sources of a sparse conv: per segment a fresh-row map and a cache-pixel map (2-D, box
// {64, 1}); row coordinate = t * rows_per_step + row.
struct GatherMaps {
    CUtensorMap fresh[2], cache[2];
    int fresh_rps[2], cache_rps[2];
};
constexpr int STG_BYTES = 8 * 16 * 32 * 2;  // (reserved: the former per-warp V^T transpose tiles)
constexpr int LAG = 2;
constexpr int GATHER_WARPS = 2;  // A warps issuing TMA gather4 in the gather mode; the rest use cp.async  // cp.async stages in flight per A-producer thread
constexpr int SEL_BYTES = BM * 19 * 4;  // select-on-read table [128][18] + row pixels [128]

struct Layout {
    int bn, stage, stages, total;
};

__host__ __device__ inline Layout layout(int bn) {
    Layout l;
    l.bn = bn;
    l.stage = A_BYTES + bn * BK * 2;
    l.stages = SMEM_BUDGET / l.stage;
    if (l.stages > MAX_STAGES) l.stages = MAX_STAGES;
    // stages + barriers (2 per stage + 4) + TMEM slot + epilogue tables (6 x BN floats) +
    // per-row select-on-read table (128 rows x 2 segments x 9 taps) + align
    l.total = l.stages * l.stage + 1024 + 256 + 6 * bn * 4 + SEL_BYTES + STG_BYTES + 64;
    return l;
}

FIS_DEV void tma2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
FIS_DEV void tma4d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
FIS_DEV void tma_gather4(uint32_t dst, const void* tmap, int c, int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tmap), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
FIS_DEV void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FIS_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
FIS_DEV void tmem_ld16(uint32_t taddr, uint32_t* u) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
}
FIS_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
FIS_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// debug timeline (FIS_BIG_DBG & 4): CTA 0's per-stage times [role][iteration] (%globaltimer ns)
__device__ unsigned long long g_big_trace[3][256];
FIS_DEV unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ int* g_dbg_host = nullptr;
// mbarrier wait with a watchdog (FIS_BIG_DBG & 16): report the stuck role and trap
FIS_DEV void wait_dbg(uint64_t* b, uint32_t parity, int dbg, int role, int it) {
    if (!(dbg & 16)) { mbar_wait(b, parity); return; }
    if (g_dbg_host && threadIdx.x % 32 == 0) {  // heartbeat: last wait entered per (cta < 4, role)
        if (blockIdx.x < 4) ((volatile int*)g_dbg_host)[8 * 4000 + blockIdx.x * 8 + role] = it + 1;
    }
    const unsigned long long t0 = gtime();
    for (long long n = 0;; n++) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        if ((n & 255) == 0 && gtime() - t0 > 2000000000ull && g_dbg_host) {
            // report once per (cta, role) into host-mapped memory and keep waiting
            volatile int* h = g_dbg_host + 8 * ((blockIdx.x * 8 + role) % 4096);
            if (h[0] == 0) {
                h[1] = blockIdx.x; h[2] = threadIdx.x; h[3] = role; h[4] = it; h[5] = (int)parity;
                __threadfence_system();
                h[0] = 1;
                __threadfence_system();
            }
        }
    }
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_big_kernel(const fis_gemm_args a, const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_a2,
                    const __grid_constant__ GatherMaps gm, int bn, int amode, int dbg) {
    const int ls = ltr_begin(4);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // align by pointer arithmetic on the shared array (keeps the shared address space: LDS/STS)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const Layout L = layout(bn);
    uint64_t* full = (uint64_t*)(smem + L.stages * L.stage);
    uint64_t* empty = full + L.stages;
    uint64_t* acc_full = empty + L.stages;  // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2]
    uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
    float* tabs = (float*)(smem + L.stages * L.stage + 256);
    int* seltab = (int*)(tabs + 6 * bn);
    int* rowtab = seltab + BM * 18;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_n = (a.n + bn - 1) / bn, tiles_m = (a.m + BM - 1) / BM;
    const int ntiles = tiles_m * tiles_n;
    const int kblocks = (a.k + BK - 1) / BK;
    // tile width bn <= 512: nsub MMAs of bns columns per K block; two TMEM accumulators when they fit
    const int nsub = bn > 256 ? 2 : 1, bns = bn / nsub, nbuf = 2 * bn <= 512 ? 2 : 1;

    if (tid == 0) {
        for (int s = 0; s < L.stages; s++) {
            mbar_init(full + s, amode == A_CPASYNC      ? A_WARPS * 32 + 1
                                : amode == A_TMA_GATHER ? GATHER_WARPS * 8 + (A_WARPS - GATHER_WARPS) * 32 + 1
                                                        : 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, amode == A_TMA_ROWS || amode == A_TMA_CONV ? 256 : 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == B_WARP && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_b) : "memory");
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int t = cur_step(a.step);  // host-written before the step: safe to read before the wait
    pdl_trigger();
    pdl_wait();
    ltr(ls, 2);

    if (warp < A_WARPS) {
        if (amode != A_CPASYNC && amode != A_TMA_GATHER) goto epilogue_role;  // TMA stages A: help the epilogue
        // ------------------------------------------------------------ A producers
        // Row metadata: thread tid resolves tile row tid (pixel, and for CONV the select-on-read
        // decision of every tap) into shared tables. Loads: lane l copies 16-byte chunk l & 7 of
        // rows w*32 + 4*i + (l >> 3), i = 0..7, so each warp instruction reads four whole 128-byte
        // rows (coalesced) and writes them conflict-free into the swizzled stage.
        const char* abase = a.a.ptr ? ref_base(a.a, t) : nullptr;
        const char* f0 = a.nsrc > 0 && a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
        const char* c0p = a.nsrc > 0 && a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
        const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
        const char* c1p = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
        const bool conv = a.a_mode == FIS_A_CONV3X3;
        const long long ldf0 = a.src[0].fresh.ld, ldc0 = a.src[0].cache.ld;
        const long long ldf1 = a.src[1].fresh.ld, ldc1 = a.src[1].cache.ld;
        const long long lda = a.a.ld;
        const int src0c = a.nsrc > 0 ? a.src[0].c : 0;
        const int cin = conv ? src0c + (a.nsrc > 1 ? a.src[1].c : 0) : a.k;
        const uint32_t sbase = smem_u32(smem);
        const char* dummy = (const char*)a.b.ptr;
        const int j = lane & 7, rbase = warp * 32 + (lane >> 3);
        int it = 0;
        int last_m = -1;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int mt = tile / tiles_n;
            if (mt != last_m) {  // row metadata once per M tile
                last_m = mt;
                const int r = mt * BM + tid;
                const bool valid = r < a.m;
                const int p = valid ? (a.rows ? __ldg(a.rows + r) : r) : -1;
                rowtab[tid] = p;
                if (conv) {
                    int* sel = seltab + tid * 18;
                    if (valid) {
                        build_sel(a, p, 0, sel);
                        if (a.nsrc > 1) build_sel(a, p, 1, sel + 9);
                    } else {
#pragma unroll
                        for (int q = 0; q < 18; q++) sel[q] = SEL_ZERO;
                    }
                }
                __syncwarp();
            }
            if (amode == A_TMA_GATHER) {
                // lanes 0-7 of each warp own 4-row groups: one TMA gather4 per group and K block when
                // the 4 rows come from one source (fresh rows / cached pixels, zero padding = OOB
                // row); a group mixing both sources is copied with cp.async (mask borders only)
                // (hybrid: warps < GATHER_WARPS issue gather4 for their rows, the other A warps
                // copy theirs with cp.async, so the TMA unit and the LSU work in parallel)
                const int g0 = 4 * (warp * 8 + lane);
                for (int kb = 0; kb < kblocks; kb++, it++) {
                    const int s = it % L.stages;
                    if (it >= L.stages) wait_dbg(empty + s, ((it / L.stages) & 1) ^ 1, dbg, 0, it);
                    if ((dbg & 4) && blockIdx.x == 0 && tid == 0 && it < 256) g_big_trace[0][it] = gtime();
                    if (warp >= GATHER_WARPS) {
                        const int k0 = kb * BK, tap = k0 / cin;
                        int c = k0 - tap * cin;
                        const int seg = c >= src0c ? 1 : 0;
                        c -= seg ? src0c : 0;
                        const char* fb = (seg ? f1 : f0) + (c + j * 8) * 2;
                        const char* cb = (seg ? c1p : c0p) + (c + j * 8) * 2;
                        const long long ldf = (seg ? ldf1 : ldf0) * 2, ldc = (seg ? ldc1 : ldc0) * 2;
                        const int* selc = seltab + rbase * 18 + seg * 9 + tap;
                        int v[8];
#pragma unroll
                        for (int i = 0; i < 8; i++) v[i] = selc[i * 4 * 18];
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            const char* src = v[i] == SEL_ZERO ? nullptr
                                              : v[i] >= 0      ? fb + (long long)v[i] * ldf
                                                               : cb + (long long)(-2 - v[i]) * ldc;
                            cp_async16(sbase + s * L.stage + sw128_off(rbase + 4 * i, j),
                                       src ? (const void*)src : (const void*)dummy, src != nullptr);
                        }
                        cp_async_arrive_noinc(full + s);
                    } else if (lane < 8) {
                        const int k0 = kb * BK, tap = k0 / cin;
                        int c = k0 - tap * cin;
                        const int seg = c >= src0c ? 1 : 0;
                        c -= seg ? src0c : 0;
                        int v[4], nf = 0, nc = 0;
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            v[i] = seltab[(g0 + i) * 18 + seg * 9 + tap];
                            nf += v[i] >= 0;
                            nc += v[i] <= -2 && v[i] != SEL_ZERO;
                        }
                        const uint32_t dst = sbase + s * L.stage + g0 * 128;
                        if (nc == 0 || nf == 0) {
                            const bool fr = nc == 0;
                            const int base = t * (fr ? gm.fresh_rps[seg] : gm.cache_rps[seg]);
                            int rr[4];
#pragma unroll
                            for (int i = 0; i < 4; i++)
                                rr[i] = v[i] == SEL_ZERO ? -1 : base + (fr ? v[i] : -2 - v[i]);
                            arrive_expect_tx(full + s, 4 * 128);
                            tma_gather4(dst, fr ? (seg ? &gm.fresh[1] : &gm.fresh[0]) : (seg ? &gm.cache[1] : &gm.cache[0]),
                                        c, rr[0], rr[1], rr[2], rr[3], full + s);
                        } else {
                            const char* fb = (seg ? f1 : f0) + c * 2;
                            const char* cb = (seg ? c1p : c0p) + c * 2;
                            const long long ldf = (seg ? ldf1 : ldf0) * 2, ldc = (seg ? ldc1 : ldc0) * 2;
#pragma unroll
                            for (int i = 0; i < 4; i++) {
                                const char* src = v[i] == SEL_ZERO ? nullptr
                                                  : v[i] >= 0      ? fb + (long long)v[i] * ldf
                                                                   : cb + (long long)(-2 - v[i]) * ldc;
#pragma unroll
                                for (int q = 0; q < 8; q++)
                                    cp_async16(sbase + s * L.stage + sw128_off(g0 + i, q),
                                               src ? (const void*)(src + q * 16) : (const void*)dummy, src != nullptr);
                            }
                            cp_async_arrive_noinc(full + s);
                        }
                    }
                }
                continue;
            }
            // rows mode: this thread's 8 row pointers for the whole tile
            const char* rp[8];
            if (!conv) {
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int p = rowtab[rbase + 4 * i];
                    rp[i] = p >= 0 ? abase + (long long)p * lda * 2 + j * 16 : nullptr;
                }
            }
            for (int kb = 0; kb < kblocks; kb++, it++) {
                const int s = it % L.stages;
                if (it >= L.stages) wait_dbg(empty + s, ((it / L.stages) & 1) ^ 1, dbg, 0, it);
                if ((dbg & 4) && blockIdx.x == 0 && tid == 0 && it < 256) g_big_trace[0][it] = gtime();
                const int k0 = kb * BK;
                const uint32_t sa = sbase + s * L.stage;
                const char* src[8];
                if (conv) {
                    const int tap = k0 / cin;
                    int c = k0 - tap * cin;
                    const int seg = c >= src0c ? 1 : 0;
                    c -= seg ? src0c : 0;
                    const char* fb = (seg ? f1 : f0) + (c + j * 8) * 2;
                    const char* cb = (seg ? c1p : c0p) + (c + j * 8) * 2;
                    const long long ldf = (seg ? ldf1 : ldf0) * 2, ldc = (seg ? ldc1 : ldc0) * 2;
                    const int* selc = seltab + rbase * 18 + seg * 9 + tap;
                    int v[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) v[i] = selc[i * 4 * 18];  // 8 independent shared loads
#pragma unroll
                    for (int i = 0; i < 8; i++)
                        src[i] = v[i] == SEL_ZERO ? nullptr
                                 : v[i] >= 0      ? fb + (long long)v[i] * ldf
                                                  : cb + (long long)(-2 - v[i]) * ldc;
                } else {
                    const bool kok = k0 + j * 8 < a.k && !(dbg & 2);
#pragma unroll
                    for (int i = 0; i < 8; i++) src[i] = rp[i] && kok ? rp[i] + k0 * 2 : nullptr;
                }
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const bool ok = src[i] != nullptr && !(dbg & 2);
                    cp_async16(sa + sw128_off(rbase + 4 * i, j), ok ? (const void*)src[i] : (const void*)dummy, ok);
                }
                if (dbg & 8) {
                    cp_async_arrive_noinc(full + s);
                } else {
                    // keep LAG stages of this thread's copies in flight; publish the oldest one
                    cp_commit();
                    if (it >= LAG) {
                        cp_wait<LAG>();
                        fence_async_smem();
                        mbar_arrive(full + (it - LAG) % L.stages);
                    }
                }
            }
        }
        if (!(dbg & 8) && amode == A_CPASYNC) {  // drain: publish the last LAG stages
            cp_wait<0>();
            fence_async_smem();
            for (int q = it - LAG < 0 ? 0 : it - LAG; q < it; q++) mbar_arrive(full + q % L.stages);
        }
    } else if (warp == B_WARP) {
        // ------------------------------------------------------------ B producer (TMA)
        if (lane == 0) {
            const uint32_t sbase = smem_u32(smem);
            // A bytes are expected here only when this thread also issues the A tile (rows / dense conv);
            // gather lanes expect their own 4-row bytes
            const uint32_t bbytes = (uint32_t)(bn * BK * 2) + (amode == A_TMA_ROWS || amode == A_TMA_CONV ? A_BYTES : 0);
            // TMA A geometry: 128 consecutive output pixels = a box of whole image rows (hw >= 128)
            // or of whole images (hw < 128); 3x3 taps are shifted boxes, padding = TMA zero fill
            const int ow = a.out_w, ohw = a.out_h * a.out_w;
            const int cin0 = a.nsrc > 0 ? a.src[0].c : 0, cin = cin0 + (a.nsrc > 1 ? a.src[1].c : 0);
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int n0 = (tile % tiles_n) * bn, m0 = (tile / tiles_n) * BM;
                const int img = amode == A_TMA_CONV ? m0 / ohw : 0;
                const int y0 = amode == A_TMA_CONV && ohw >= BM ? (m0 - img * ohw) / ow : 0;
                for (int kb = 0; kb < kblocks; kb++, it++) {
                    const int s = it % L.stages;
                    if (it >= L.stages) wait_dbg(empty + s, ((it / L.stages) & 1) ^ 1, dbg, 1, it);
                    if ((dbg & 4) && blockIdx.x == 0 && it < 256) g_big_trace[1][it] = gtime();
                    arrive_expect_tx(full + s, bbytes);
                    const uint32_t sa = sbase + s * L.stage;
                    for (int j = 0; j < nsub; j++)
                        tma2d(sa + A_BYTES + j * bns * 128, &tmap_b, kb * BK, n0 + j * bns, full + s);
                    if (amode == A_TMA_ROWS) {
                        tma2d(sa, &tmap_a, kb * BK, m0, full + s);
                    } else if (amode == A_TMA_CONV) {
                        const int k0 = kb * BK, tap = k0 / cin;
                        int c = k0 - tap * cin;
                        const bool seg1 = c >= cin0;
                        c -= seg1 ? cin0 : 0;
                        tma4d(sa, seg1 ? &tmap_a2 : &tmap_a, c, tap % 3 - 1, y0 + tap / 3 - 1, img, full + s);
                    }
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bns >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);
        const uint32_t sbase = smem_u32(smem);
        int it = 0, lt = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, lt++) {
            const int buf = lt % nbuf, use = lt / nbuf;
            if (use >= 1) wait_dbg(acc_empty + buf, (use & 1) ^ 1, dbg, 2, lt);  // epilogue drained this buffer
            tc_fence_after();
            const uint32_t dt = tmem + buf * ACC_STRIDE;
            for (int kb = 0; kb < kblocks; kb++, it++) {
                const int s = it % L.stages;
                wait_dbg(full + s, (it / L.stages) & 1, dbg, 3, it);
                tc_fence_after();
                if ((dbg & 4) && blockIdx.x == 0 && lane == 0 && it < 256) g_big_trace[2][it] = gtime();
                if (lane == 0) {
                    const uint32_t sa = sbase + s * L.stage, sb = sa + A_BYTES;
                    for (int j = 0; j < nsub; j++) {  // tiles wider than 256: one MMA per 128 x bns half
#pragma unroll
                        for (int kk = 0; kk < BK / 16; kk++) {
                            const uint64_t ad = sw128_desc(sa + kk * 32), bd = sw128_desc(sb + j * bns * 128 + kk * 32);
                            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt + j * bns),
                                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        }
                    }
                    mma_commit(empty + s);
                    if (kb == kblocks - 1) mma_commit(acc_full + buf);
                }
                __syncwarp();
            }
        }
    } else {
        goto epilogue_role;
    }
    goto teardown;
epilogue_role : {
        // ------------------------------------------------------------ epilogue
        // warps 6-9 (group 0); with TMA-staged A the idle warps 0-3 join as group 1 and the two
        // groups take alternate 16-column chunks of every tile
        const int nepi = amode == A_TMA_ROWS || amode == A_TMA_CONV ? 256 : 128;
        const int grp = warp < A_WARPS ? 1 : 0;
        const int et = grp ? tid + 128 : tid - EPI_WARP0 * 32;  // 0..nepi-1
        const int quarter = warp & 3;         // TMEM lane quarter this warp may access
        const int lr = quarter * 32 + lane;   // tile row of this thread
        const int cstep = nepi == 256 ? 2 : 1;
        const EpiCtx e = make_epi(a, t);
        // fast row stores: bf16 row-major d (16-byte aligned rows), epilogue = bias (+ residual) only;
        // same arithmetic as row_epilogue (alpha == 1: v * 1 is exact)
        const bool fast = a.epi == FIS_EPI_NONE && a.alpha == 1.0f && !e.pre && !e.pre2 && !e.bias2 && !e.lat &&
                          !a.d_rows && !a.d_trans && a.d.dtype == FIS_BF16 && (a.d.ld % 8) == 0 &&
                          (((uintptr_t)e.d) & 15) == 0 && (!e.res || (a.res.ld % 8) == 0);
        // transposed V^T of a fused QKV (n >= n_split) through the staging tile
        const bool tfast = fast && !e.res && a.n_split > 0 && a.d2_trans && a.d2.dtype == FIS_BF16 &&
                           (a.d2.ld % 8) == 0 && (((uintptr_t)e.d2) & 15) == 0 && !(dbg & 1);
        EpiTab tb;
        tb.mean = tabs;
        tb.rstd = tb.mean + bn;
        tb.bias = tb.rstd + bn;
        tb.b2 = tb.bias + bn;
        tb.gamma = tb.b2 + bn;
        tb.beta = tb.gamma + bn;
        int lt = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, lt++) {
            const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * bn;
            named_sync(1, nepi);  // previous tile's table reads done
            for (int c = et; c < bn; c += nepi) {
                const int n = n0 + c;
                const bool ok = n < a.n;
                tb.bias[c] = ok && a.bias ? __ldg(a.bias + n) : 0.f;
                tb.b2[c] = ok && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n) : 0.f;
                if (a.epi == FIS_EPI_GN_SILU && ok) {
                    const int g = n / e.cpg;
                    const float rstd = (float)(1.0 / sqrt((double)e.var[g] + (double)a.eps));
                    const float scale = rstd * __ldg(a.gamma + n);
                    tb.mean[c] = scale;
                    tb.rstd[c] = fmaf(-e.mean[g], scale, __ldg(a.beta + n));
                } else {
                    tb.mean[c] = 0.f;
                    tb.rstd[c] = 0.f;
                }
            }
            named_sync(1, nepi);
            const int buf = lt % nbuf;
            wait_dbg(acc_full + buf, (lt / nbuf) & 1, dbg, 4, lt);
            tc_fence_after();
            const uint32_t taddr = tmem + buf * ACC_STRIDE + ((uint32_t)(quarter * 32) << 16);
            const int r = m0 + lr;
            for (int cb = 16 * grp; cb < bn; cb += 16 * cstep) {
                uint32_t u[16];
                tmem_ld16(taddr + cb, u);
                tmem_wait_ld();
                const int nn = n0 + cb;
                if (tfast && nn >= a.n_split && nn + 16 <= a.n) {
                    // transposed V^T chunk (fused QKV): V^T[dn + j][r] -- for each j the warp's 32 rows
                    // are 64 contiguous bytes: direct 2-byte stores, coalesced per j (a shared-memory
                    // transpose round trip measured slower on the CTA-pair kernel: L0 QKV 36 -> 28.5 us)
                    if (r < a.m) {
                        __nv_bfloat16* dst = (__nv_bfloat16*)e.d2 + (long long)(nn - a.n_split) * a.d2.ld + r;
#pragma unroll
                        for (int j = 0; j < 16; j++)
                            dst[(long long)j * a.d2.ld] = __float2bfloat16_rn(__fadd_rn(__uint_as_float(u[j]), tb.bias[cb + j]));
                    }
                    continue;
                }
                if (r < a.m && !(dbg & 1)) {
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 16; j++) v[j] = __uint_as_float(u[j]);
                    const int n = n0 + cb;
                    if (fast && n + 16 <= (a.n_split > 0 ? a.n_split : a.n)) {
                        // plain bf16 row store (+ bias, + residual): no per-chunk mode dispatch
#pragma unroll
                        for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], tb.bias[cb + j]);
                        if (e.res) {
                            float q[16];
                            load_row16(e.res, a.res.dtype, (long long)r * a.res.ld + n, 16, q);
#pragma unroll
                            for (int j = 0; j < 16; j++) v[j] = __fadd_rn(v[j], q[j]);
                        }
                        uint4 o[2];
                        __nv_bfloat162* h = (__nv_bfloat162*)o;
#pragma unroll
                        for (int j = 0; j < 8; j++) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                        uint4* dp = (uint4*)((__nv_bfloat16*)e.d + (long long)r * a.d.ld + n);
                        dp[0] = o[0];
                        dp[1] = o[1];
                    } else {
                        row_epilogue_any(a, e, tb, r, cb, n0, v);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty + buf);
        }
    }
teardown:
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace big
}  // namespace fis

// ---------------------------------------------------------------------------- host side

namespace {

// Weight tensor maps, cached by (base, n, k, ld, box): a captured step re-encodes nothing.
struct MapEntry {
    const void* base;
    long long n, k, ld;
    int box;
    CUtensorMap map;
};
constexpr int MAP_CACHE = 512;
MapEntry g_maps[MAP_CACHE];
int g_nmaps = 0, g_next = 0;

const CUtensorMap* weight_map(const void* base, long long n, long long k, long long ld, int box) {
    for (int i = 0; i < g_nmaps; i++) {
        const MapEntry& m = g_maps[i];
        if (m.base == base && m.n == n && m.k == k && m.ld == ld && m.box == box) return &m.map;
    }
    MapEntry e{base, n, k, ld, box, {}};
    if (!encode_2d(&e.map, base, n, k, ld, box)) return nullptr;
    int slot;
    if (g_nmaps < MAP_CACHE) slot = g_nmaps++;
    else { slot = g_next; g_next = (g_next + 1) % MAP_CACHE; }
    g_maps[slot] = e;
    return &g_maps[slot].map;
}

}  // namespace

const CUtensorMap* fis_weight_map(const void* base, long long n, long long k, long long ld, int box) {
    return weight_map(base, n, k, ld, box);
}

namespace {

int sms() {
    static int n = 0;
    if (n <= 0) n = fis_device_sm_count();
    return n > 0 ? n : 148;
}

}  // namespace

// Tile width: the largest multiple of 16 in [128, 256] dividing N; else 256 (or N rounded up
// to 16 when N < 256).
int fis_gemm_big_bn(int n) {
    static int force = getenv("FIS_BIG_BN") ? atoi(getenv("FIS_BIG_BN")) : 0;
    if (force) return force;
    for (int bn = 256; bn >= 128; bn -= 16)
        if (n % bn == 0) return bn;
    if (n < 256) return (n + 15) & ~15;
    return 256;
}

static bool tma_a_ok(const fis_gemm_args* a);
static bool gather_ok(const fis_gemm_args* a);

// The persistent kernel takes GEMMs whose tile count fills the SMs (stacked requests): bf16 A
// (gathered rows or 3x3 conv), static bf16 weights addressable by TMA, no split-K. With TMA-staged
// A (dense maps / contiguous rows) it beats the per-op kernel from ~40 tiles on.
int fis_gemm_big_eligible(const fis_gemm_args* a) {
    if (getenv("FIS_BIG") && getenv("FIS_BIG")[0] == '0') return 0;
    if (a->splits > 1 || a->n < 128 || a->b.step_stride != 0) return 0;
    const int bn = fis_gemm_big_bn(a->n);
    const long long tiles = (long long)((a->m + 127) / 128) * ((a->n + bn - 1) / bn);
    static long long min_tiles = getenv("FIS_BIG_MIN_TILES") ? atoll(getenv("FIS_BIG_MIN_TILES")) : -1;
    if (min_tiles >= 0) return tiles >= min_tiles ? 1 : 0;
    // gathered (cp.async) A: the per-op kernel's 2-threads-per-row gather is as fast (r01 probe)
    if (tiles >= 40 && tma_a_ok(a)) return 1;
    return tiles >= 100 && gather_ok(a) ? 1 : 0;  // TMA gather4 pays off from ~100 tiles (r01 probe)
}

// 4-D bf16 map of a dense stacked source [img][h][w][c] (pixel stride ld), box {64, w, bh, bi}
// covering 128 consecutive pixels.
static bool encode_conv4(CUtensorMap* out, const fis_src& s, long long images) {
    const int hw = s.h * s.w;
    int bh, bi;
    if (hw >= 128) {
        if (128 % s.w || hw % 128) return false;
        bh = 128 / s.w;
        bi = 1;
    } else {
        if (128 % hw) return false;
        bh = s.h;
        bi = 128 / hw;
    }
    if (s.w > 256 || bh > 256 || (((uintptr_t)s.fresh.ptr) & 15) || (s.fresh.ld % 8) || s.fresh.ld < s.c) return false;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const long long rb = s.fresh.ld * 2;
    cuuint64_t dims[4] = {(cuuint64_t)s.c, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)images};
    cuuint64_t strides[3] = {(cuuint64_t)rb, (cuuint64_t)(rb * s.w), (cuuint64_t)(rb * hw)};
    cuuint32_t box[4] = {64u, (cuuint32_t)s.w, (cuuint32_t)bh, (cuuint32_t)bi};
    cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    return enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(s.fresh.ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool conv_box_ok(const fis_src& s) {
    const int hw = s.h * s.w;
    if (hw >= 128) return 128 % s.w == 0 && hw % 128 == 0 && s.w <= 256;
    return 128 % hw == 0;
}

static bool tma_a_ok(const fis_gemm_args* a) {
    static int off = getenv("FIS_BIG_TMA_A") && getenv("FIS_BIG_TMA_A")[0] == '0';
    if (off || a->rows) return false;
    if (a->a_mode == FIS_A_ROWS) return !a->a.step_stride && a->a.dtype == FIS_BF16 && (a->a.ld % 8) == 0;
    const int hw = a->out_h * a->out_w;
    if (hw <= 0 || a->m % hw) return false;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.index || s.up || s.fresh.step_stride || s.fresh.dtype != FIS_BF16 || s.h != a->out_h ||
            s.w != a->out_w || !conv_box_ok(s) || (s.fresh.ld % 8))
            return false;
    }
    return true;
}

// TMA staging of A when every source is a plain bf16 matrix without per-step stride: contiguous
// rows (ROWS, no row list) or dense 3x3 conv sources at the output resolution (no select-on-read,
// no upsampling, no row list).
static int choose_amode(const fis_gemm_args* a, CUtensorMap* ta, CUtensorMap* ta2) {
    if (!tma_a_ok(a)) return fis::big::A_CPASYNC;
    if (a->a_mode == FIS_A_ROWS) {
        if (a->a.step_stride || a->a.dtype != FIS_BF16) return fis::big::A_CPASYNC;
        return encode_2d(ta, a->a.ptr, a->m, a->k, a->a.ld, 128) ? fis::big::A_TMA_ROWS : fis::big::A_CPASYNC;
    }
    const int hw = a->out_h * a->out_w;
    if (hw <= 0 || a->m % hw) return fis::big::A_CPASYNC;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.index || s.up || s.fresh.step_stride || s.fresh.dtype != FIS_BF16 || s.h != a->out_h || s.w != a->out_w)
            return fis::big::A_CPASYNC;
        if (!encode_conv4(i ? ta2 : ta, s, a->m / hw)) return fis::big::A_CPASYNC;
    }
    if (a->nsrc < 2) *ta2 = *ta;
    return fis::big::A_TMA_CONV;
}

// Sparse convs (select-on-read over compact fresh rows + the cached slab): TMA gather4 per source.
static bool gather_ok(const fis_gemm_args* a) {
    static int off = getenv("FIS_BIG_GATHER") && getenv("FIS_BIG_GATHER")[0] == '0';
    if (off || a->a_mode != FIS_A_CONV3X3) return false;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (s.fresh.dtype != FIS_BF16 || (s.fresh.ld % 8) || (((uintptr_t)s.fresh.ptr) & 15) ||
            (s.fresh.step_stride % (s.fresh.ld * 2)))
            return false;
        if (s.index && (s.cache.dtype != FIS_BF16 || (s.cache.ld % 8) || (((uintptr_t)s.cache.ptr) & 15) ||
                        (s.cache.step_stride % (s.cache.ld * 2))))
            return false;
    }
    return true;
}

static bool encode_gather(const fis_gemm_args* a, fis::big::GatherMaps* gm) {
    const long long huge = 1ll << 30;
    for (int i = 0; i < a->nsrc; i++) {
        const fis_src& s = a->src[i];
        if (!encode_2d(&gm->fresh[i], s.fresh.ptr, huge, s.c, s.fresh.ld, 1)) return false;
        gm->fresh_rps[i] = (int)(s.fresh.step_stride / (s.fresh.ld * 2));
        if (s.index) {
            if (!encode_2d(&gm->cache[i], s.cache.ptr, huge, s.c, s.cache.ld, 1)) return false;
            gm->cache_rps[i] = (int)(s.cache.step_stride / (s.cache.ld * 2));
        } else {
            gm->cache[i] = gm->fresh[i];
            gm->cache_rps[i] = gm->fresh_rps[i];
        }
    }
    if (a->nsrc < 2) {
        gm->fresh[1] = gm->fresh[0];
        gm->cache[1] = gm->cache[0];
        gm->fresh_rps[1] = gm->fresh_rps[0];
        gm->cache_rps[1] = gm->cache_rps[0];
    }
    return true;
}

// Gathered A is the expensive operand: one tile covers up to 512 output columns (two MMAs per K
// block, single accumulator) so each gathered row is loaded once per 320-512 columns.
static int wide_bn(int n) {
    static int off = getenv("FIS_BIG_WIDE") && getenv("FIS_BIG_WIDE")[0] == '0';
    if (off) return 0;
    for (int bn = 512; bn > 256; bn -= 32)
        if (n % bn == 0 && (bn / 2) % 16 == 0) return bn;
    return 0;
}

// TMA staging of A for the per-op kernel (fis_gemm_tc.cu): 0 none, 1 contiguous rows, 2 dense conv
int fis_tma_a_encode(const fis_gemm_args* a, CUtensorMap* ta, CUtensorMap* ta2) {
    return choose_amode(a, ta, ta2);
}

static long long g_big_launched = 0;
// persistent-kernel launches so far (tests check that fis_gemm did not fall back to the per-op kernel)
extern "C" long long fis_gemm_big_launch_count(void) { return g_big_launched; }

int fis_gemm_big_launch(const fis_gemm_args* a, cudaStream_t stream) {
    CUtensorMap ta, ta2;
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&ta2, 0, sizeof(ta2));
    int amode = choose_amode(a, &ta, &ta2);
    static fis::big::GatherMaps gm;  // kernel parameter copy; static keeps it off the stack
    std::memset(&gm, 0, sizeof(gm));
    static int gmode = getenv("FIS_BIG_GATHER") ? atoi(getenv("FIS_BIG_GATHER")) : 1;  // 2: cp.async gather
    if (amode == fis::big::A_CPASYNC && gmode == 1 && gather_ok(a) && encode_gather(a, &gm))
        amode = fis::big::A_TMA_GATHER;
    int bn = fis_gemm_big_bn(a->n);
    static int wide_off = getenv("FIS_BIG_WIDE") && getenv("FIS_BIG_WIDE")[0] == '0';
    if ((amode == fis::big::A_CPASYNC || amode == fis::big::A_TMA_GATHER) && !wide_off) {
        const int w = wide_bn(a->n);
        if (w) bn = w;
    } else if (!wide_off && !getenv("FIS_BIG_BN")) {
        // TMA-staged A: a 320-wide tile (two N = 160 MMAs per K block) when it needs fewer waves
        // of tiles x tile width (e.g. 4096 x 1280: 160 tiles of 256 = 2 waves on 148 SMs, 128
        // tiles of 320 = 1 wave)
        const int w = wide_bn(a->n);
        if (w) {
            const long long mt = (a->m + 127) / 128;
            const long long t0 = mt * ((a->n + bn - 1) / bn), t1 = mt * ((a->n + w - 1) / w);
            const long long c0 = (t0 + sms() - 1) / sms() * bn, c1 = (t1 + sms() - 1) / sms() * w;
            if (c1 < c0) bn = w;
        }
    }
    const CUtensorMap* tm = weight_map(a->b.ptr, a->n, a->k, a->b.ld, bn > 256 ? bn / 2 : bn);
    if (!tm) return FIS_ERR_UNSUPPORTED;
    const fis::big::Layout L = fis::big::layout(bn);
    static int configured_smem = 0;
    if (configured_smem < L.total) {
        // dynamic + static shared memory must fit the 227 KB per-block limit
        cudaFuncAttributes fa;
        const int stat = cudaFuncGetAttributes(&fa, fis::big::gemm_big_kernel) == cudaSuccess ? (int)fa.sharedSizeBytes : 1024;
        const int maxdyn = 227 * 1024 - stat;
        if (L.total > maxdyn ||
            cudaFuncSetAttribute(fis::big::gemm_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxdyn) !=
                cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured_smem = maxdyn;
    }
    const long long tiles = (long long)((a->m + 127) / 128) * ((a->n + bn - 1) / bn);
    const int grid = (int)(tiles < sms() ? tiles : sms());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(fis::big::THREADS);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fis_pdl_enabled() ? 1 : 0;
    static int dbg = getenv("FIS_BIG_DBG") ? atoi(getenv("FIS_BIG_DBG")) : 0;  // 1: no stores, 2: no A loads
    if (cudaLaunchKernelEx(&cfg, fis::big::gemm_big_kernel, *a, *tm, ta, ta2, gm, bn, amode, dbg) != cudaSuccess)
        return FIS_ERR_LAUNCH;
    g_big_launched++;
    return FIS_OK;
}

extern "C" int fis_big_trace_read(unsigned long long* out768) {
    return cudaMemcpyFromSymbol(out768, fis::big::g_big_trace, sizeof(fis::big::g_big_trace)) == cudaSuccess
               ? FIS_OK : FIS_ERR_LAUNCH;
}

extern "C" int fis_big_debug_buf(int* host_mapped) {
    return cudaMemcpyToSymbol(fis::big::g_dbg_host, &host_mapped, sizeof(int*)) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}

FIS_LTR_SETTER(fis_ltr_set_big)
