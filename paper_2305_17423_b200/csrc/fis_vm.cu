// Persistent step VM for sm_100a: one CTA per SM runs a whole recorded UNet step.
//
// The host records the launches of one step (Engine.run_step in capture mode) as a list of
// fis_vm_op records; fis_vm_plan tiles them and fis_vm_run executes them in ONE launch:
//
//   op j, item i  ->  CTA (cta0_j + i) mod G          (cta0 rotates from op to op)
//   an item of op j waits until op dep_j (the previous non-empty op) has completed all of
//   its items (a device-scope counter per op, release/acquire), so the step's ~100 ops run
//   back to back with no launch gap, no per-kernel prologue (barrier init, TMEM alloc) and
//   no tail; a CTA whose next item is a GEMM stages that item's weight (B) tiles into its
//   shared-memory ring BEFORE the dependency resolves — weights do not depend on the
//   previous op — so the weight stream of op j+1 overlaps op j.
//
// Warp roles (288 threads) as in the per-op tcgen05 GEMM (fis_gemm_tc.cu):
//   warps 0-7 : producers (A gather with select-on-read, B weight rows; 16-byte cp.async into
//               SW128 K-major stages) and the epilogue (tcgen05.ld -> fused row epilogue);
//               they also run the SIMT ops (softmax, GN stats/apply, pool, SIMT GEMM).
//   warp 8    : MMA issuer; walks the same op list and consumes the smem ring.
// The ring, its phase and the TMEM accumulator persist across items and ops.
// Split-K partials go to a workspace; the last-arriving CTA of a tile sums them in split
// order (bitwise deterministic) and runs the epilogue.
#define FIS_LOADS_CG 1  // every element load of this translation unit bypasses L1 (see fis_common.cuh)
#include "fis_tc.cuh"

namespace fis {
namespace vm {
using namespace fis::tc;

#ifndef VM_STAGES
#define VM_STAGES 4
#endif
#ifndef VM_MIN_SPLIT_KB
#define VM_MIN_SPLIT_KB 16  // K blocks below which a GEMM is not split (split items keep >= half of it)
#endif
#ifndef VM_FUSED_ATTN
#define VM_FUSED_ATTN 1
#endif
// warps 0-3 producers / epilogue, warp 4 idle, warp 5 MMA (its spin-waits share an SM sub-partition
// with warp 1, not with warp 0 whose thread 0 issues the TMA loads).  6 warps are allocated
// registers like 8, so each thread may use 255 registers (no spills in the fused paths).
constexpr int STAGES = VM_STAGES, PRODUCERS = 128, THREADS = 192, MMA_WARP = 5;
constexpr int TPR = PRODUCERS / 128;   // producer threads per 128-byte smem row of a stage
constexpr int CPT = 8 / TPR;           // 16-byte chunks each of them loads per row
constexpr int WPQ = PRODUCERS / 128;   // epilogue warps per TMEM lane quarter
constexpr int MAX_BN = 128;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = MAX_BN * BK * 2;
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int OPBUF = 1024;
constexpr int EPI = MAX_BN * 32;
constexpr int SEL = BM * 2 * 9 * 4;
constexpr int RES_LD = 272;                  // bytes per staged residual row (<= 256 B of data)
constexpr int RES_BYTES = VM_FUSED_ATTN ? BM * RES_LD : 0;  // epilogue operand tile (residual / latent rows)
constexpr int P_BYTES = VM_FUSED_ATTN ? 2 * BM * 64 * 2 : 0;  // attention P tile: 128 x 128 keys bf16 (two SW128 chunks)
constexpr int TMEM_COLS = 512;
constexpr int SMEM = STAGES * STAGE + RES_BYTES + P_BYTES + 1024;  // dynamic: ring + operand tile + P (+ align)
constexpr int ELEMS_PER_ITEM = 2048;  // elementwise ops
constexpr int SOFTMAX_ROWS = PRODUCERS / 32;  // one warp per row
constexpr int SBM = 64, SBN = 64, SBK = 64;  // SIMT GEMM tile (64-deep k passes: all gathers of a pass in flight)

static_assert(sizeof(fis_vm_op) <= OPBUF, "fis_vm_op must fit the shared op buffer");

FIS_DEV void pbar() { asm volatile("bar.sync 1, %0;" ::"n"(PRODUCERS) : "memory"); }

// 2^x on the SFU (bf16-mode softmax: scores are pre-scaled by scale * log2(e))
FIS_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// the step index of this launch (read once per CTA from fis_vm_args.step)
__shared__ int s_step;

FIS_DEV int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct Shared {
    unsigned char* ring;
    unsigned char* res;  // staged epilogue operand rows [BM][RES_LD]
    unsigned char* pbuf; // attention P tile
    uint64_t* s_ready;   // attention: every S block of the item is in TMEM
    uint64_t* p_ready;   // attention: P block written (256 producer arrivals)
    uint64_t* p_free;    // attention: the P.V MMAs reading the P tile have completed
    uint64_t* red;       // split-K: the split partial slices of this CTA's rows have landed
    fis_vm_op* op;
    EpiTab tb;
    int* seltab;
    uint64_t* full;
    uint64_t* empty;
    uint64_t* done;
    uint32_t* tmem_slot;
    int* flag;
};

// Shared-memory layout: the ring (dynamic, 1024-aligned) and static shared objects, so every
// pointer below stays in the shared address space (LDS/STS, no generic loads, no aliasing
// with global stores).
extern __shared__ __align__(1024) unsigned char vm_smem[];
__shared__ __align__(16) fis_vm_op s_op;
__shared__ __align__(16) float s_tab[6][MAX_BN];
__shared__ __align__(16) int s_sel[BM * 2 * 9];
__shared__ __align__(8) uint64_t s_bar[2 * STAGES + 5];
__shared__ __align__(16) fis_gemm_args s_ea;   // attention: epilogue view (out = res + O)
__shared__ __align__(16) float s_rowstat[WPQ][BM];           // attention: per-row partial max / sum of the key halves
__shared__ uint32_t s_tmem;
__shared__ int s_flag;

FIS_DEV Shared carve() {
    Shared s;
    const uint32_t a = smem_u32(vm_smem);
    s.ring = vm_smem + ((1024u - (a & 1023u)) & 1023u);
    s.res = s.ring + STAGES * STAGE;
    s.pbuf = s.res + RES_BYTES;
    s.op = &s_op;
    s.tb.mean = s_tab[0];
    s.tb.rstd = s_tab[1];
    s.tb.bias = s_tab[2];
    s.tb.b2 = s_tab[3];
    s.tb.gamma = s_tab[4];
    s.tb.beta = s_tab[5];
    s.seltab = s_sel;
    s.full = s_bar;
    s.empty = s_bar + STAGES;
    s.done = s_bar + 2 * STAGES;
    s.s_ready = s_bar + 2 * STAGES + 1;
    s.p_ready = s_bar + 2 * STAGES + 2;
    s.p_free = s_bar + 2 * STAGES + 3;
    s.red = s_bar + 2 * STAGES + 4;
    s.tmem_slot = &s_tmem;
    s.flag = &s_flag;
    return s;
}

// Shared-memory objects by constant address (nothing to keep in registers): the 1024-aligned
// ring inside the dynamic allocation and an epilogue-table view of s_tab.
FIS_DEV unsigned char* vm_ring() {
    const uint32_t a = smem_u32(vm_smem);
    return vm_smem + ((1024u - (a & 1023u)) & 1023u);
}
FIS_DEV EpiTab vm_tab() {
    EpiTab t;
    t.mean = s_tab[0]; t.rstd = s_tab[1]; t.bias = s_tab[2]; t.b2 = s_tab[3]; t.gamma = s_tab[4]; t.beta = s_tab[5];
    return t;
}

// ---------------------------------------------------------------------------------- GEMM geometry
struct GemmItem {
    int z, tile, n0, m0, kb0, nk, bn;
};

FIS_DEV GemmItem gemm_item(const fis_vm_op& op, int i) {
    GemmItem g;
    const int S = op.splits;
    g.z = i % S;
    g.tile = i / S;
    const int tn = g.tile % op.tiles_n, tm = g.tile / op.tiles_n;
    g.bn = op.bn;
    g.n0 = tn * op.bn;
    g.m0 = tm * BM;
    const int kblocks = (op.u.gemm.k + BK - 1) / BK;
    const int per = (kblocks + S - 1) / S;
    g.kb0 = g.z * per;
    g.nk = max(0, min(kblocks, g.kb0 + per) - g.kb0);
    return g;
}

// Attention item i: query tile x value slice. S block j (<= 128 keys) lives in TMEM columns
// [128 j, 128 j + N_j), the O slice in [TMEM_COLS - dvs, TMEM_COLS).
struct AttnItem {
    int m0, c0, dvs, nkb, dch, o_col;
};

FIS_DEV AttnItem attn_item(const fis_vm_op& op, int i) {
    AttnItem g;
    g.dvs = op.bn;
    g.m0 = (i / op.tiles_n) * BM;
    g.c0 = (i % op.tiles_n) * op.bn;
    g.nkb = (op.u.attn.n_keys + 127) / 128;
    g.dch = op.u.attn.d / 64;
    g.o_col = TMEM_COLS - op.bn;
    return g;
}
FIS_DEV int attn_nb(int n_keys, int j) { return min(128, n_keys - 128 * j); }

FIS_DEV uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

FIS_DEV void mma4(uint32_t d, uint32_t sa, uint32_t sb, uint32_t idesc, bool accumulate) {
#pragma unroll
    for (int kk = 0; kk < BK / 16; kk++) {
        const uint64_t ad = sw128_desc(sa + kk * 32), bd = sw128_desc(sb + kk * 32);
        const uint32_t acc = (accumulate || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
}

// TMA: 2D tile of a tensor map (box {64 elems, rows}, SW128) into shared memory; completion is
// counted in bytes on the stage's full barrier
FIS_DEV void tma2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
FIS_DEV void tma3d(uint32_t dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// expect bytes without arriving (a later arrive completes the phase)
FIS_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// arrive when this thread's prior cp.async land; the pending count is incremented now
FIS_DEV void cp_async_arrive_inc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// mbarrier wait with a sleep back-off (waiting producers leave issue slots to the TMA / MMA threads)
FIS_DEV void mbar_wait_backoff(uint64_t* b, uint32_t parity, int ns = 128) {
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
    }
}
FIS_DEV void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FIS_DEV const void* tmap_at(const fis_vm_args& va, int idx) {
    return idx >= 0 ? (const void*)((const char*)va.tmaps + 128 * (long long)idx) : nullptr;
}

FIS_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

FIS_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------------- MMA warp
FIS_DEV void mma_role(const fis_vm_args& va, const Shared& sh, uint32_t tmem, int lane) {
    const int G = gridDim.x, cta = blockIdx.x;
    uint32_t it = 0, pb = 0;
    const uint32_t sbase = smem_u32(vm_ring());
    for (int j = 0; j < va.n_ops; j++) {
        const fis_vm_op* op = va.ops + j;
        if (op->kind == FIS_VM_ATTN) {
            for (int i = (cta - op->cta0 + G) % G; i < op->n_items; i += G) {
                const AttnItem g = attn_item(*op, i);
                const int n_keys = op->u.attn.n_keys;
                for (int jb = 0; jb < g.nkb; jb++) {  // S_j = Q K_j^T
                    const uint32_t id = idesc_f16(BM, (attn_nb(n_keys, jb) + 15) & ~15);
                    for (int kc = 0; kc < g.dch; kc++, it++) {
                        const int s = it % STAGES;
                        mbar_wait(s_bar + s, (it / STAGES) & 1);
                        tc_fence_after();
                        if (lane == 0) {
                            const uint32_t sa = sbase + s * STAGE;
                            mma4(tmem + 128 * jb, sa, sa + A_BYTES, id, kc > 0);
                            mma_commit((s_bar + STAGES) + s);
                        }
                        __syncwarp();
                    }
                }
                if (lane == 0) mma_commit((s_bar + 2 * STAGES + 1));
                __syncwarp();
                const uint32_t ido = idesc_f16(BM, g.dvs), pbase = smem_u32((vm_ring() + STAGES * STAGE + RES_BYTES));
                for (int jb = 0; jb < g.nkb; jb++, pb++) {  // O += P_j V_j
                    mbar_wait((s_bar + 2 * STAGES + 2), pb & 1);
                    tc_fence_after();
                    const int nch = (attn_nb(n_keys, jb) + 63) / 64;
                    for (int c = 0; c < nch; c++, it++) {
                        const int s = it % STAGES;
                        mbar_wait(s_bar + s, (it / STAGES) & 1);
                        tc_fence_after();
                        if (lane == 0) {
                            mma4(tmem + g.o_col, pbase + c * (BM * 128), sbase + s * STAGE + A_BYTES, ido, jb > 0 || c > 0);
                            mma_commit((s_bar + STAGES) + s);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) mma_commit((s_bar + 2 * STAGES + 3));
                    __syncwarp();
                }
                if (lane == 0) mma_commit((s_bar + 2 * STAGES));
                __syncwarp();
            }
            continue;
        }
        if (op->kind != FIS_VM_GEMM || op->impl != 2) continue;
        const int n_items = op->n_items;
        const bool traced = va.trace_items && j == va.trace_op && lane == 0;
        for (int i = (cta - op->cta0 + G) % G; i < n_items; i += G) {
            const GemmItem g = gemm_item(*op, i);
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(g.bn >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
            if (traced) va.trace_items[16 * i + 14] = gtimer();
            for (int q = 0; q < g.nk; q++, it++) {
                const int s = it % STAGES;
                mbar_wait(s_bar + s, (it / STAGES) & 1);
                if (traced && q == 0) va.trace_items[16 * i + 12] = gtimer();
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sa = sbase + s * STAGE, sb = sa + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; kk++) {
                        const uint64_t ad = sw128_desc(sa + kk * 32), bd = sw128_desc(sb + kk * 32);
                        const uint32_t acc = (q > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32((s_bar + STAGES) + s))
                                 : "memory");
                }
                __syncwarp();
            }
            if (lane == 0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32((s_bar + 2 * STAGES)))
                             : "memory");
            if (traced) va.trace_items[16 * i + 13] = gtimer();
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------------- producers
FIS_DEV void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t u[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] = __uint_as_float(u[j]);
}

struct ProdState {
    uint32_t it;      // ring slot sequence number (matches the MMA warp)
    uint32_t items;   // tcgen05 items run (parity of the done barrier)
    uint32_t attn;    // attention items run (parity of s_ready)
    uint32_t pb;      // attention P blocks written (parity of p_ready / p_free, matches the MMA warp)
    uint32_t red;     // split-K reductions run (parity of the red barrier)
};


// phase stamp of item i of the traced op (profiling; fis_vm_args.trace_op / trace_items)
#define VM_STAMP(slot)                                                                   \
    do {                                                                                 \
        if (va.trace_items && j == va.trace_op && tid == 0) va.trace_items[16 * i + (slot)] = gtimer(); \
    } while (0)

FIS_DEV void trace_start(const fis_vm_args& va, int j, int tid) {
    if (va.trace && tid == 0) atomicMin(va.trace + 2 * j, gtimer());
}

// Wait (once per op) until op.dep has completed. Relaxed polling (no per-poll L1
// invalidation), then one gpu-scope fence: acquire + this SM's L1 invalidated once.
FIS_DEV int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

FIS_DEV void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Consumer side of an op dependency: relaxed polling, no acquire fence -- a gpu-scope acquire
// invalidates the whole L1 (CCTL.IVALL), which would turn every later load of static data
// (weights, index lists, op records) into an L2 round trip.  Instead every read of data produced
// inside the launch bypasses L1 (ld.global.cg, cp.async.cg, TMA, bulk copies), and the producer
// publishes with a release reduction after its stores.
FIS_DEV void spin_until(const int* c, int target, int ns) {
    while (ld_relaxed(c) < target) __nanosleep(ns);
}

FIS_DEV void red_release_add(int* c, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(c), "r"(v) : "memory");
}

FIS_DEV void wait_dep(const fis_vm_args& va, const fis_vm_op& op, int j, bool& waited, int tid) {
    if (waited) return;
    waited = true;
    if (op.dep < 0) {
        trace_start(va, j, tid);
        return;
    }
    if (tid == 0) {
        spin_until(va.sync + 1 + op.dep, op.dep_target, va.poll_ns > 0 ? va.poll_ns : 32);
        // the operands were written through the generic proxy; thread 0 reads them with TMA
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    trace_start(va, j, tid);
    pbar();
}

FIS_DEV void signal_done(const fis_vm_args& va, int j, int tid) {
    pbar();
    if (tid == 0) {
        red_release_add(va.sync + 1 + j, 1);
        if (va.trace) atomicMax(va.trace + 2 * j + 1, gtimer());
    }
}

FIS_DEV void issue_b(const fis_gemm_args& a, const GemmItem& g, const char* bbase, uint32_t sb, int k0, int ar,
                     int j0) {
    if (ar >= g.bn) return;
    const int bn = g.n0 + ar;
    const char* brow = bbase + (long long)bn * a.b.ld * 2;
#pragma unroll
    for (int j = j0; j < j0 + CPT; j++) {
        const bool ok = bn < a.n && k0 + j * 8 < a.k;
        cp_async16(sb + sw128_off(ar, j), ok ? (const void*)(brow + (k0 + j * 8) * 2) : (const void*)bbase, ok);
    }
}

// Per-column epilogue parameters of the tile (bias, time bias, cached GN stats, gamma/beta).
FIS_DEV void stage_tables(const fis_gemm_args& a, const EpiCtx& e, const Shared& sh, int n0, int bn, int tid) {
    for (int c = tid; c < bn; c += PRODUCERS) {
        const int n = n0 + c;
        const bool ok = n < a.n;
        vm_tab().bias[c] = ok && a.bias ? __ldg(a.bias + n) : 0.f;
        vm_tab().b2[c] = ok && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n) : 0.f;
        if (a.epi == FIS_EPI_GN_SILU && ok) {
            const int gi = n / e.cpg;
            // cached-stat GN folded into one fma per element: y = v * scale + shift
            const float rstd = (float)(1.0 / sqrt((double)e.var[gi] + (double)a.eps));
            const float scale = rstd * __ldg(a.gamma + n);
            vm_tab().mean[c] = scale;
            vm_tab().rstd[c] = fmaf(-e.mean[gi], scale, __ldg(a.beta + n));
            vm_tab().gamma[c] = 0.f;
            vm_tab().beta[c] = 0.f;
        } else {
            vm_tab().mean[c] = 0.f; vm_tab().rstd[c] = 0.f; vm_tab().gamma[c] = 0.f; vm_tab().beta[c] = 0.f;
        }
    }
}

// 8 consecutive elements of one row: vector access when aligned (16 B bf16 / 2x16 B f32)
FIS_DEV void load8(const char* base, int dtype, long long off, int nvalid, float* v) {
    if (dtype == FIS_BF16) {
        const __nv_bfloat16* p = (const __nv_bfloat16*)base + off;
        if (nvalid == 8 && ((uintptr_t)p & 15) == 0) {
            const uint4 u = FIS_LD_U4(p);
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const float2 f = __bfloat1622float2(h[k]);
                v[2 * k] = f.x; v[2 * k + 1] = f.y;
            }
            return;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) if (k < nvalid) v[k] = load_elem((const char*)p, FIS_BF16, k);
    } else {
        const float* p = (const float*)base + off;
        if (nvalid == 8 && ((uintptr_t)p & 15) == 0) {
            const float4 a0 = FIS_LD_F4(p), a1 = FIS_LD_F4(p + 4);
            v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
            return;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) if (k < nvalid) v[k] = load_elem((const char*)p, FIS_F32, k);
    }
}

FIS_DEV void store8(char* base, int dtype, long long off, int nvalid, const float* v) {
    if (dtype == FIS_BF16) {
        __nv_bfloat16* p = (__nv_bfloat16*)base + off;
        if (nvalid == 8 && ((uintptr_t)p & 15) == 0) {
            uint4 u;
            __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
            *(uint4*)p = u;
            return;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) if (k < nvalid) p[k] = __float2bfloat16_rn(v[k]);
    } else {
        float* p = (float*)base + off;
        if (nvalid == 8 && ((uintptr_t)p & 15) == 0) {
            *(float4*)p = make_float4(v[0], v[1], v[2], v[3]);
            *(float4*)(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
            return;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) if (k < nvalid) p[k] = v[k];
    }
}

// Fused GEMM epilogue of 8 columns of one output row; same operations in the same order as
// fis::tc::row_epilogue (fis_tc.cuh) so the VM and the per-op kernels agree. Split in two so a
// thread can issue the global reads (residual, latent rows) of several items before using them.
struct EpiIn {
    float x[8];  // latent rows (EPI_STEP) or residual (the plan rejects GEMMs with both)
};

FIS_DEV void epilogue8_load(const fis_gemm_args& a, const EpiCtx& e, int r, int n, EpiIn& in,
                            const unsigned char* staged_row) {
    const int nvalid = min(8, a.n - n);
    if (staged_row) {  // rows staged in shared memory by stage_operand
        const int dtype = a.epi == FIS_EPI_STEP ? a.lat.dtype : a.res.dtype;
        if (dtype == FIS_BF16) {
            const uint4 u = *(const uint4*)staged_row;
            const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const float2 f = __bfloat1622float2(h[k]);
                in.x[2 * k] = f.x; in.x[2 * k + 1] = f.y;
            }
        } else {
            const float4 a0 = *(const float4*)staged_row, a1 = *(const float4*)(staged_row + 16);
            in.x[0] = a0.x; in.x[1] = a0.y; in.x[2] = a0.z; in.x[3] = a0.w;
            in.x[4] = a1.x; in.x[5] = a1.y; in.x[6] = a1.z; in.x[7] = a1.w;
        }
        return;
    }
    const int orow = a.d_rows ? __ldg(a.d_rows + r) : r;
    if (a.epi == FIS_EPI_STEP) load8(e.lat, a.lat.dtype, (long long)orow * a.lat.ld + n, nvalid, in.x);
    else if (e.res) load8(e.res, a.res.dtype, (long long)orow * a.res.ld + n, nvalid, in.x);
}

FIS_DEV void epilogue8(const fis_gemm_args& a, const EpiCtx& e, const EpiTab& tb, int r, int c0, int n0, float* v,
                       const EpiIn& in) {
    const int n = n0 + c0;
    const int nvalid = min(8, a.n - n);
    const int orow = a.d_rows ? __ldg(a.d_rows + r) : r;
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k] * a.alpha, tb.bias[c0 + k]);
    if (e.pre) store8(e.pre, a.pre.dtype, (long long)orow * a.pre.ld + n, nvalid, v);
    if (e.bias2) {
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k], tb.b2[c0 + k]);
    }
    if (a.epi == FIS_EPI_GN_SILU) {
        float y[8];
#pragma unroll
        for (int k = 0; k < 8; k++)
            y[k] = fmaf(v[k], tb.mean[c0 + k], tb.rstd[c0 + k]);  // scale / shift (stage_tables)
        if (e.pre2) store8(e.pre2, a.pre2.dtype, (long long)orow * a.pre2.ld + n, nvalid, y);
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __fdividef(y[k], 1.0f + __expf(-y[k]));
    } else if (a.epi == FIS_EPI_STEP) {
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __fsub_rn(in.x[k], __fmul_rn(a.step_scale, v[k]));
    }
    if (e.res && a.epi != FIS_EPI_STEP) {
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k], in.x[k]);
    }
    char* dbase = e.d;
    int dt = a.d.dtype, dld = a.d.ld, dn = n, trans = a.d_trans;
    if (a.n_split > 0 && n >= a.n_split) {  // fused QKV: V part goes transposed to d2
        dbase = e.d2; dt = a.d2.dtype; dld = a.d2.ld; dn = n - a.n_split; trans = a.d2_trans;
    }
    if (trans) {
#pragma unroll
        for (int k = 0; k < 8; k++) if (k < nvalid) store_elem(dbase, dt, (long long)(dn + k) * dld + orow, v[k]);
    } else {
        store8(dbase, dt, (long long)orow * dld + dn, nvalid, v);
    }
}

template <int BN>
FIS_DEV void gemm_tc_epilogue(const fis_vm_args& va, const Shared& sh, int j, int i,
                                              const GemmItem& g, ProdState& ps, uint32_t tmem, int tid,
                                              bool tables_done, bool staged);

// The epilogue's one read operand of this tile (latent rows for EPI_STEP, else the residual):
// rows [m0, m0+BM) x columns [n0, n0+bn) copied to (vm_ring() + STAGES * STAGE) with 16-byte cp.async when the row
// segment fits RES_LD and is 16-byte aligned.  Returns false (direct loads) otherwise.
FIS_DEV bool stage_operand(const fis_gemm_args& a, const Shared& sh, const GemmItem& g, int t, int tid) {
    if (RES_BYTES == 0) return false;
    const fis_ref& x = a.epi == FIS_EPI_STEP ? a.lat : a.res;
    if (!x.ptr || a.d_rows) return false;
    const int esz = x.dtype == FIS_BF16 ? 2 : 4;
    const int ncols = min(g.bn, a.n - g.n0);
    const int seg = ((ncols * esz) + 15) & ~15;
    if (seg > RES_LD || (ncols * esz) % 16 || ((long long)x.ld * esz) % 16 || ((long long)g.n0 * esz) % 16) return false;
    const char* base = ref_base(x, t) + (long long)g.n0 * esz;
    if (((uintptr_t)base) & 15) return false;
    const int per_row = seg / 16;
    const int rows = min(BM, a.m - g.m0);
    const uint32_t dst0 = smem_u32((vm_ring() + STAGES * STAGE));
    for (int idx = tid; idx < rows * per_row; idx += PRODUCERS) {
        const int row = idx / per_row, c16 = idx % per_row;
        const int col_bytes = c16 * 16;
        const char* src = base + ((long long)(g.m0 + row) * x.ld) * esz + col_bytes;
        cp_async16(dst0 + row * RES_LD + col_bytes, src, true);
    }
    cp_commit();
    return true;
}

template <int BN>
FIS_DEV void gemm_tc_item(const fis_vm_args& va, const Shared& sh, int j, int i, ProdState& ps,
                                          bool& waited, uint32_t tmem, int tid) {
    const fis_vm_op& op = s_op;
    const fis_gemm_args& a = op.u.gemm;
    const GemmItem g = gemm_item(op, i);
    const int t = s_step;
    const int ar = tid / TPR, half_id = tid % TPR, j0 = half_id * CPT;
    const uint32_t sbase = smem_u32(vm_ring());
    const char* bbase = ref_base(a.b, t);

    VM_STAMP(0);
    // Ring protocol: each slot's full barrier expects ONE arrival (thread 0) plus the TMA bytes;
    // cp.async loads register themselves with incrementing cp.async.mbarrier.arrive before a
    // producer barrier that precedes thread 0's arrival.  TMA-only k-blocks are issued by
    // thread 0 alone; the other producers go straight to the epilogue.
    // ---- weight tiles of the first stages + static epilogue tables: independent of the previous
    //      op when B is static (weights / per-edit text K/V)
    if (!op.b_static) wait_dep(va, op, j, waited, tid);
    const void* tma_b = tmap_at(va, op.tmap_b);
    const void* tma_a = tmap_at(va, op.tmap_a);
    const void* tma_a2 = tmap_at(va, op.tmap_a2);
    const bool conv = a.a_mode == FIS_A_CONV3X3;
    const int cin = conv ? a.src[0].c + (a.nsrc > 1 ? a.src[1].c : 0) : a.k;
    const int src0c = a.nsrc > 0 ? a.src[0].c : 0;
    // k-block q takes A from a TMA map?
    auto a_map = [&](int k0) -> const void* {
        if (!conv) return tma_a;
        const int c = k0 % cin;
        return c >= src0c ? tma_a2 : tma_a;
    };
    const uint32_t b_bytes = (uint32_t)(BK * BN * 2);
    const int npre = min(g.nk, STAGES);
    if (tma_b) {
        if (tid == 0)
            for (int q = 0; q < npre; q++) {
                const uint32_t sq = ps.it + q;
                const int s = sq % STAGES;
                if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                mbar_expect_tx(s_bar + s, b_bytes);
                tma2d(sbase + s * STAGE + A_BYTES, tma_b, (g.kb0 + q) * BK, g.n0, s_bar + s);
            }
    } else {
        for (int q = 0; q < npre; q++) {
            const uint32_t sq = ps.it + q;
            const int s = sq % STAGES;
            if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
            issue_b(a, g, bbase, sbase + s * STAGE + A_BYTES, (g.kb0 + q) * BK, ar, j0);
        }
    }
    if (op.b_static) stage_tables(a, make_epi(a, t), sh, g.n0, g.bn, tid);
    // ---- static gather metadata (row/index lists are fixed for the whole edit)
    const int r = g.m0 + ar;
    const bool row_valid = r < a.m;
    const int row_p = row_valid ? (a.rows ? __ldg(a.rows + r) : r) : 0;
    if (conv)
        for (int seg = half_id; seg < a.nsrc; seg += TPR) build_sel(a, row_p, seg, s_sel + (ar * 2 + seg) * 9);
    __syncwarp();  // the two threads of a row each built one segment's select table
    VM_STAMP(1);
    wait_dep(va, op, j, waited, tid);
    VM_STAMP(2);

    const char* abase = a.a.ptr ? ref_base(a.a, t) : nullptr;
    const char* f0 = a.nsrc > 0 && a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
    const char* c0p = a.nsrc > 0 && a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
    const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
    const char* c1p = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
    const int* mysel = s_sel + ar * 2 * 9;
    const bool mixed = conv && a.nsrc > 1 && ((tma_a != nullptr) != (tma_a2 != nullptr));
    for (int q = 0; q < g.nk; q++) {
        const uint32_t sq = ps.it + q;
        const int s = sq % STAGES;
        const uint32_t sa = sbase + s * STAGE;
        const int k0 = (g.kb0 + q) * BK;
        const void* tm = tma_b ? a_map(k0) : nullptr;  // TMA A only together with TMA B
        if (tm && mixed) {
            // ---- conv with one TMA segment and one gathered segment: every producer stays in step
            if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
            if (tid == 0) {
                if (q >= npre) {
                    mbar_expect_tx(s_bar + s, b_bytes);
                    tma2d(sa + A_BYTES, tma_b, k0, g.n0, s_bar + s);
                }
                const int tap = k0 / cin;
                const int c = k0 - tap * cin;
                const int cs = c >= src0c ? c - src0c : c;
                mbar_expect_tx(s_bar + s, (uint32_t)(BM * BK * 2));
                tma3d(sa, tm, cs, tap % 3 - 1, g.m0 / a.out_w + tap / 3 - 1, s_bar + s);
            }
            pbar();
            if (tid == 0) mbar_arrive(s_bar + s);
            continue;
        }
        if (tm) {
            // ---- thread 0 alone: (B if not prefetched) + A via TMA, one arrival with the bytes
            if (tid == 0) {
                if (q >= npre) {
                    mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                    mbar_expect_tx(s_bar + s, b_bytes);
                    tma2d(sa + A_BYTES, tma_b, k0, g.n0, s_bar + s);
                }
                expect_tx(s_bar + s, (uint32_t)(BM * BK * 2));
                if (conv) {
                    const int tap = k0 / cin;
                    const int c = k0 - tap * cin;
                    const int cs = c >= src0c ? c - src0c : c;
                    tma3d(sa, tm, cs, tap % 3 - 1, g.m0 / a.out_w + tap / 3 - 1, s_bar + s);
                } else {
                    tma2d(sa, tm, k0, g.m0, s_bar + s);
                }
                if (q == 0) VM_STAMP(8);
            }
            continue;
        }
        // ---- every producer: gathered A rows (and B rows without TMA) with cp.async; every thread
        //      waits for the slot itself (only thread 0 waited for the TMA-prefetched B stages)
        if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
        if (q >= npre) {
            if (tma_b) {
                if (tid == 0) {
                    mbar_expect_tx(s_bar + s, b_bytes);
                    tma2d(sa + A_BYTES, tma_b, k0, g.n0, s_bar + s);
                }
            } else {
                issue_b(a, g, bbase, sa + A_BYTES, k0, ar, j0);
            }
        }
        const char* src = nullptr;
        if (row_valid) {
            if (a.a_mode == FIS_A_ROWS) {
                if (k0 < a.k) src = abase + ((long long)row_p * a.a.ld + k0) * 2;
            } else {
                const int tap = k0 / cin;
                int c = k0 - tap * cin;
                const int seg = c >= src0c ? 1 : 0;
                c -= seg ? src0c : 0;
                const int sel = mysel[seg * 9 + tap];
                if (sel != SEL_ZERO) {
                    const fis_src& sr = a.src[seg];
                    if (sel >= 0) src = (seg ? f1 : f0) + ((long long)sel * sr.fresh.ld + c) * 2;
                    else src = (seg ? c1p : c0p) + ((long long)(-2 - sel) * sr.cache.ld + c) * 2;
                }
            }
        }
#pragma unroll
        for (int jj = j0; jj < j0 + CPT; jj++) {
            const bool ok = src != nullptr && (conv || k0 + jj * 8 < a.k);
            cp_async16(sa + sw128_off(ar, jj), ok ? (const void*)(src + jj * 16) : (const void*)bbase, ok);
        }
        cp_async_arrive_inc(s_bar + s);
        pbar();  // every producer's arrival is registered before thread 0's
        if (tid == 0) mbar_arrive(s_bar + s);
        if (q == 0) VM_STAMP(8);
    }
    ps.it += g.nk;
    // ---- epilogue operand rows (residual, or latent rows for the step update): produced by
    //      earlier ops, so fetched now into shared memory, landing while the MMAs run
    const bool staged = stage_operand(a, sh, g, t, tid);
    VM_STAMP(3);
    gemm_tc_epilogue<BN>(va, sh, j, i, g, ps, tmem, tid, op.b_static != 0, staged);
}

// Fast epilogue (bf16 row-major output, no recording stores): thread -> one 8-column chunk,
// rows strided by PRODUCERS / (BN/8); bias / time-bias / GN parameters of its 8 columns are
// loaded once into registers; accumulators come from the staging tile (S == 1) or the split
// partials (S > 1, summed in split order); the residual / latent rows from the staged operand.
template <int BN, int MODE>
FIS_DEV void fast_epilogue(const fis_gemm_args& a, const EpiCtx& e, const Shared& sh, const GemmItem& g,
                           const float* stage, const float* wsb, long long tile_floats, int S, int r0, int nrows,
                           bool staged, int tid) {
    constexpr int CH = BN / 8, RSTEP = PRODUCERS / CH, PLD = BN + 4;
    const int ch = tid % CH, cb = ch * 8, n = g.n0 + cb;
    if (n >= a.n) return;
    const int nvalid = min(8, a.n - n);
    // column parameters stay in shared memory (re-read per row: two 16-byte LDS each) so the
    // row loop needs no extra registers
    auto ld8 = [&](const float* t, float* o) {
        const float4 x0 = *(const float4*)(t + cb), x1 = *(const float4*)(t + cb + 4);
        o[0] = x0.x; o[1] = x0.y; o[2] = x0.z; o[3] = x0.w; o[4] = x1.x; o[5] = x1.y; o[6] = x1.z; o[7] = x1.w;
    };
    const float alpha = a.alpha, step_scale = a.step_scale;
    const bool has_b2 = e.bias2 != nullptr, has_x = staged;
    const int xdt = MODE == FIS_EPI_STEP ? a.lat.dtype : a.res.dtype;
    const int xesz = xdt == FIS_BF16 ? 2 : 4;
    __nv_bfloat16* dst = (__nv_bfloat16*)e.d + n;
    const int dld = a.d.ld;
    for (int rr = tid / CH; rr < nrows; rr += RSTEP) {
        const int row = r0 + rr;
        float v[8];
        if (S == 1) {
            const float4 f0 = *(const float4*)(stage + row * PLD + cb);
            const float4 f1 = *(const float4*)(stage + row * PLD + cb + 4);
            v[0] = f0.x; v[1] = f0.y; v[2] = f0.z; v[3] = f0.w; v[4] = f1.x; v[5] = f1.y; v[6] = f1.z; v[7] = f1.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = 0.f;
            const float* p = wsb + row * BN + cb;
            int zz = 0;
            for (; zz + 3 <= S; zz += 3) {  // 6 float4 loads in flight, summed in split order
                float4 f[3][2];
#pragma unroll
                for (int q = 0; q < 3; q++)
#pragma unroll
                    for (int w = 0; w < 2; w++) f[q][w] = *((const float4*)(p + (zz + q) * tile_floats) + w);
#pragma unroll
                for (int q = 0; q < 3; q++)
#pragma unroll
                    for (int w = 0; w < 2; w++) {
                        v[4 * w] += f[q][w].x; v[4 * w + 1] += f[q][w].y;
                        v[4 * w + 2] += f[q][w].z; v[4 * w + 3] += f[q][w].w;
                    }
            }
            for (; zz < S; zz++) {
#pragma unroll
                for (int w = 0; w < 2; w++) {
                    const float4 f = *((const float4*)(p + zz * tile_floats) + w);
                    v[4 * w] += f.x; v[4 * w + 1] += f.y; v[4 * w + 2] += f.z; v[4 * w + 3] += f.w;
                }
            }
        }
        float x[8];
        if (has_x) {
            const unsigned char* xr = (vm_ring() + STAGES * STAGE) + row * RES_LD + cb * xesz;
            if (xdt == FIS_BF16) {
                const uint4 u = *(const uint4*)xr;
                const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const float2 f = __bfloat1622float2(h[k]);
                    x[2 * k] = f.x; x[2 * k + 1] = f.y;
                }
            } else {
                const float4 a0 = *(const float4*)xr, a1 = *(const float4*)(xr + 16);
                x[0] = a0.x; x[1] = a0.y; x[2] = a0.z; x[3] = a0.w; x[4] = a1.x; x[5] = a1.y; x[6] = a1.z; x[7] = a1.w;
            }
        }
        // same operations, same order as fis::tc::row_epilogue
        {
            float t8[8];
            ld8(vm_tab().bias, t8);
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k] * alpha, t8[k]);
            if (has_b2) {
                ld8(vm_tab().b2, t8);
#pragma unroll
                for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k], t8[k]);
            }
        }
        if (MODE == FIS_EPI_GN_SILU) {
            float gs[8], gh[8];
            ld8(vm_tab().mean, gs);
            ld8(vm_tab().rstd, gh);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const float y = fmaf(v[k], gs[k], gh[k]);
                v[k] = __fdividef(y, 1.0f + __expf(-y));
            }
        } else if (MODE == FIS_EPI_STEP) {
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = __fsub_rn(x[k], __fmul_rn(step_scale, v[k]));
        }
        if (MODE != FIS_EPI_STEP && has_x) {
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = __fadd_rn(v[k], x[k]);
        }
        __nv_bfloat16* p = dst + (long long)(g.m0 + row) * dld;
        if (nvalid == 8) {
            uint4 u;
            __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
            for (int k = 0; k < 4; k++) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
            *(uint4*)p = u;
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) if (k < nvalid) p[k] = __float2bfloat16_rn(v[k]);
        }
    }
}

// Epilogue of one tcgen05 GEMM item (separate frame: the gather pointers above are dead here).
//   1. TMEM -> shared staging tile [BM][BN+4] fp32 (thread = accumulator row)
//   2. S == 1: fused row epilogue over (row, 16-column chunk) items, consecutive threads on
//      consecutive chunks of a row (full-sector coalesced loads/stores); transposed outputs use
//      consecutive threads on consecutive rows instead.
//      S > 1 : the staged partial is copied (coalesced) to the workspace; the S split CTAs of
//      the tile meet at a tile counter, then split z reduces rows [z*BM/S, (z+1)*BM/S) over
//      all S partials in split order (bitwise deterministic) and runs the epilogue on them.
//      Every split CTA of a tile is resident and co-scheduled (plan: items <= CTAs when S > 1).
template <int BN>
FIS_DEV void gemm_tc_epilogue(const fis_vm_args& va, const Shared& sh, int j, int i,
                                              const GemmItem& g, ProdState& ps, uint32_t tmem, int tid,
                                              bool tables_done, bool staged) {
    const fis_vm_op& op = s_op;
    const fis_gemm_args& a = op.u.gemm;
    const int warp = tid >> 5, lane = tid & 31;
    const int t = s_step;
    const EpiCtx e = make_epi(a, t);
    if (!tables_done) stage_tables(a, e, sh, g.n0, g.bn, tid);
    VM_STAMP(4);
    mbar_wait_backoff((s_bar + 2 * STAGES), ps.items & 1);
    ps.items++;
    tc_fence_after();
    VM_STAMP(5);
    // ---- 1. TMEM -> staging (the ring is idle: every MMA of this item has completed)
    constexpr int PLD = BN + 4;
    constexpr int hc = BN / WPQ;  // columns per warp of a lane quarter
    float* stage = (float*)vm_ring();
    {
        const int quarter = warp & 3, half = warp >> 2;  // WPQ warps share a lane quarter
        const int lr = quarter * 32 + lane;
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + half * hc;
        float* dst = stage + lr * PLD + half * hc;
#pragma unroll 1
        for (int q = 0; q < hc / 16; q++) {
            float v[16];
            tmem_ld16(taddr + 16 * q, v);
#pragma unroll
            for (int w = 0; w < 4; w++)
                *(float4*)(dst + 16 * q + 4 * w) = make_float4(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]);
        }
        tc_fence_before();
    }
    VM_STAMP(9);
    if (staged) cp_wait<0>();
    pbar();
    VM_STAMP(10);
    const int S = op.splits;
    constexpr int chunks = BN / 8;  // 8-column epilogue items
    int r0 = 0, r1 = BM;
    const float* wsb = nullptr;
    const long long tile_floats = (long long)BM * BN;
    long long tile_floats_red = tile_floats;  // stride between split partials as the reduce reads them
    if (S > 1) {
        // ---- 2b. publish the partial with bulk copies (one 512 B row per thread), meet the other
        //      splits of the tile, then bulk-load this split's rows of all S partials into smem
        float* wsz = va.ws + ((long long)g.tile * S + g.z) * tile_floats;
        if (tid < BM) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(wsz + tid * BN),
                         "r"(smem_u32(stage + tid * PLD)), "r"(BN * 4)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        pbar();
        const int rows_per = (BM + S - 1) / S;
        r0 = min(BM, g.z * rows_per);
        r1 = min(BM, r0 + rows_per);
        const int slice_floats = rows_per * BN;
        float* red = (float*)vm_ring();  // staging is free once the partial is published
        if (tid == 0) {
            int* ctr = va.sync + op.sync_base + g.tile;
            red_release_add(ctr, 1);
            spin_until(ctr, S, 32);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t bytes = (uint32_t)((r1 - r0) * BN * 4);
            if (bytes) {
                expect_tx((s_bar + 2 * STAGES + 4), bytes * S);
                const float* src0 = va.ws + (long long)g.tile * S * tile_floats + (long long)r0 * BN;
                for (int z = 0; z < S; z++)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(red + z * slice_floats)),
                        "l"(src0 + z * tile_floats), "r"(bytes), "r"(smem_u32((s_bar + 2 * STAGES + 4)))
                        : "memory");
            } else {
                mbar_arrive((s_bar + 2 * STAGES + 4));
            }
        }
        mbar_wait_backoff((s_bar + 2 * STAGES + 4), ps.red & 1, 32);
        ps.red++;
        VM_STAMP(11);
        // the reduce reads index wsb + row * BN + z * tile_floats with row in [r0, r1)
        wsb = red - r0 * BN;
        tile_floats_red = slice_floats;
    }
    // ---- 2. fused epilogue of rows [r0, r1), 8-column items
    const int nrows = min(r1, a.m - g.m0) - r0;
    const bool trans = a.d_trans || (a.n_split > 0 && g.n0 >= a.n_split);
    const int n_items = nrows > 0 ? nrows * chunks : 0;
    // fast path: thread = fixed 8-column chunk x rows strided by PRODUCERS/chunks; the column
    // parameters live in registers, operands come from shared memory
    if (!trans && !a.d_rows && (staged || (!e.res && a.epi != FIS_EPI_STEP)) && !e.pre && !e.pre2 &&
        a.d.dtype == FIS_BF16 && (a.d.ld % 8) == 0 && (((uintptr_t)e.d) & 15) == 0 && (g.n0 % 8) == 0) {
        if (a.epi == FIS_EPI_GN_SILU)
            fast_epilogue<BN, FIS_EPI_GN_SILU>(a, e, sh, g, stage, wsb, tile_floats_red, S, r0, nrows, staged, tid);
        else if (a.epi == FIS_EPI_STEP)
            fast_epilogue<BN, FIS_EPI_STEP>(a, e, sh, g, stage, wsb, tile_floats_red, S, r0, nrows, staged, tid);
        else
            fast_epilogue<BN, FIS_EPI_NONE>(a, e, sh, g, stage, wsb, tile_floats_red, S, r0, nrows, staged, tid);
        VM_STAMP(6);
        signal_done(va, j, tid);
        VM_STAMP(7);
        return;
    }
    constexpr int IB = 2;  // items per thread in flight (their global reads issued together)
    long long cy_load = 0, cy_epi = 0, cy0 = clock64();
    for (int base = tid; base < n_items; base += IB * PRODUCERS) {
        const long long c0 = clock64();
        float v[IB][8];
        EpiIn in[IB];
        int rowv[IB], cbv[IB];
#pragma unroll
        for (int u = 0; u < IB; u++) {
            const int idx = base + u * PRODUCERS;
            int row = 0, ch = 0;
            if (idx < n_items) {
                if (trans) { row = r0 + idx % nrows; ch = idx / nrows; }
                else { row = r0 + idx / chunks; ch = idx % chunks; }
            }
            rowv[u] = row;
            cbv[u] = ch * 8;
            const bool live = idx < n_items && g.n0 + ch * 8 < a.n;
            if (!live) { cbv[u] = -1; continue; }
            if (S == 1) {
                const float4 f0 = *(const float4*)(stage + row * PLD + ch * 8);
                const float4 f1 = *(const float4*)(stage + row * PLD + ch * 8 + 4);
                v[u][0] = f0.x; v[u][1] = f0.y; v[u][2] = f0.z; v[u][3] = f0.w;
                v[u][4] = f1.x; v[u][5] = f1.y; v[u][6] = f1.z; v[u][7] = f1.w;
            }
            const int esz = (a.epi == FIS_EPI_STEP ? a.lat.dtype : a.res.dtype) == FIS_BF16 ? 2 : 4;
            epilogue8_load(a, e, g.m0 + row, g.n0 + ch * 8, in[u],
                           staged ? (vm_ring() + STAGES * STAGE) + row * RES_LD + ch * 8 * esz : nullptr);
        }
        if (S > 1) {
#pragma unroll
            for (int u = 0; u < IB; u++) {
                if (cbv[u] < 0) continue;
#pragma unroll
                for (int jj = 0; jj < 8; jj++) v[u][jj] = 0.f;
                const float* p = wsb + rowv[u] * BN + cbv[u];
                int zz = 0;
                for (; zz + 4 <= S; zz += 4) {  // 8 float4 loads in flight, summed in split order
                    float4 f[4][2];
#pragma unroll
                    for (int q = 0; q < 4; q++)
#pragma unroll
                        for (int w = 0; w < 2; w++) f[q][w] = *((const float4*)(p + (zz + q) * tile_floats_red) + w);
#pragma unroll
                    for (int q = 0; q < 4; q++)
#pragma unroll
                        for (int w = 0; w < 2; w++) {
                            v[u][4 * w] += f[q][w].x; v[u][4 * w + 1] += f[q][w].y;
                            v[u][4 * w + 2] += f[q][w].z; v[u][4 * w + 3] += f[q][w].w;
                        }
                }
                for (; zz < S; zz++) {
#pragma unroll
                    for (int w = 0; w < 2; w++) {
                        const float4 f = *((const float4*)(p + zz * tile_floats_red) + w);
                        v[u][4 * w] += f.x; v[u][4 * w + 1] += f.y; v[u][4 * w + 2] += f.z; v[u][4 * w + 3] += f.w;
                    }
                }
            }
        }
        const long long c1 = clock64();
#pragma unroll
        for (int u = 0; u < IB; u++)
            if (cbv[u] >= 0) epilogue8(a, e, vm_tab(), g.m0 + rowv[u], cbv[u], g.n0, v[u], in[u]);
        cy_load += c1 - c0;
        cy_epi += clock64() - c1;
    }
    if (va.trace_items && j == va.trace_op && tid == 0) {
        va.trace_items[16 * i + 12] = cy_load;
        va.trace_items[16 * i + 13] = cy_epi;
        va.trace_items[16 * i + 14] = clock64() - cy0;
    }
    VM_STAMP(6);
    signal_done(va, j, tid);
    VM_STAMP(7);
}

// ---------------------------------------------------------------------------------- attention
// One item: out[m0:m0+128, c0:c0+dvs] = res + softmax(Q K^T * scale) V for a 128-query tile and
// a value slice (sparse.py:265-338, tensors.py:183-200, unet.py:456-457), in one CTA:
//   S_j = Q K_j^T for every 128-key block j into TMEM (keys <= 512 - dvs), exact row max / sum
//   over all blocks (thread = row half), then per block P_j = exp(S_j*scale - m) / l -> bf16
//   SW128 tile in shared memory -> O += P_j V_j on the tensor core; epilogue adds the residual.
template <int DVS>
FIS_DEV void attn_item_run(const fis_vm_args& va, const Shared& sh, int j, int i, ProdState& ps, bool& waited,
                           uint32_t tmem, int tid) {
    const fis_vm_op& op = s_op;
    const fis_attn_args& a = op.u.attn;
    const AttnItem g = attn_item(op, i);
    const int t = s_step;
    const int warp = tid >> 5, lane = tid & 31;
    const int ar = tid / TPR, j0 = (tid % TPR) * CPT;
    const uint32_t sbase = smem_u32(vm_ring());
    // epilogue view of the output: a GEMM-style epilogue over [m, dv] with the residual
    if (tid == 0) {
        fis_gemm_args& e = s_ea;
        memset(&e, 0, sizeof(e));
        e.m = a.m; e.n = a.dv; e.k = 1; e.alpha = 1.f; e.epi = FIS_EPI_NONE;
        e.res = a.res; e.pre = a.pre; e.d = a.out;
    }
    for (int c = tid; c < DVS; c += PRODUCERS) {
        vm_tab().bias[c] = 0.f; vm_tab().b2[c] = 0.f; vm_tab().mean[c] = 0.f; vm_tab().rstd[c] = 0.f;
    }
    VM_STAMP(0);
    wait_dep(va, op, j, waited, tid);  // Q, K, V^T and the residual come from earlier ops
    pbar();                            // s_ea visible
    if (va.trace_items && j == va.trace_op && tid == 0) va.trace_items[16 * i + 14] = clock64();
    GemmItem ge;
    ge.z = 0; ge.tile = 0; ge.n0 = g.c0; ge.m0 = g.m0; ge.kb0 = 0; ge.nk = 0; ge.bn = DVS;
    VM_STAMP(2);
    const char* qb = ref_base(a.q, t);
    const char* kb = ref_base(a.k, t);
    const char* vb = ref_base(a.vt, t);
    const int n_keys = a.n_keys;
    const void* tq = tmap_at(va, op.tmap_a);
    const void* tk = tmap_at(va, op.tmap_b);
    const void* tv = tmap_at(va, op.tmap_a2);
    // ---- S phase loads, key-block major: slot (jb, kc) carries Q chunk kc and K chunk (jb, kc)
    const int qr = g.m0 + ar;
    if (tq && tk) {
        if (tid == 0) {
            uint32_t sq = ps.it;
            for (int jb = 0; jb < g.nkb; jb++)
                for (int kc = 0; kc < g.dch; kc++, sq++) {
                    const int s = sq % STAGES;
                    if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                    const uint32_t sa = sbase + s * STAGE;
                    expect_tx(s_bar + s, (uint32_t)(2 * BM * BK * 2));
                    tma2d(sa, tq, kc * 64, g.m0, s_bar + s);
                    tma2d(sa + A_BYTES, tk, kc * 64, 128 * jb, s_bar + s);
                }
        }
        ps.it += g.dch * g.nkb;
    } else {
        for (int jb = 0; jb < g.nkb; jb++)
            for (int kc = 0; kc < g.dch; kc++) {
                const int key = 128 * jb + ar;
                const uint32_t sq = ps.it++;
                const int s = sq % STAGES;
                if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                const uint32_t sa = sbase + s * STAGE, sb = sa + A_BYTES;
                const char* qs = qb + ((long long)qr * a.q.ld + kc * 64) * 2;
                const char* ks = kb + ((long long)key * a.k.ld + kc * 64) * 2;
#pragma unroll
                for (int u = j0; u < j0 + CPT; u++) {
                    cp_async16(sa + sw128_off(ar, u), qr < a.m ? (const void*)(qs + 16 * u) : (const void*)qb, qr < a.m);
                    cp_async16(sb + sw128_off(ar, u), key < n_keys ? (const void*)(ks + 16 * u) : (const void*)qb,
                               key < n_keys);
                }
                cp_async_arrive_inc(s_bar + s);
                pbar();
                if (tid == 0) mbar_arrive(s_bar + s);
            }
    }
    const bool staged = stage_operand(s_ea, sh, ge, t, tid);  // residual rows, land during the MMAs
    VM_STAMP(3);
    // ---- exact softmax statistics over every key block (thread = row lr, key half hf)
    mbar_wait_backoff((s_bar + 2 * STAGES + 1), ps.attn & 1);
    ps.attn++;
    tc_fence_after();
    VM_STAMP(8);
    constexpr int KPT = 128 / WPQ;  // keys of a block handled by each thread of a row
    const int quarter = warp & 3, hf = warp >> 2, lr = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const float scale = a.scale * 1.4426950408889634f;  // exp(s*scale - m) = 2^(s*scale*log2e - m')
    float mx = -INFINITY;
    for (int jb = 0; jb < g.nkb; jb++) {
        const int k0 = 128 * jb + KPT * hf;
#pragma unroll 1
        for (int q = 0; q < KPT / 16; q++) {
            if (k0 + 16 * q >= n_keys) break;
            float v[16];
            tmem_ld16(trow + 128 * jb + KPT * hf + 16 * q, v);
#pragma unroll
            for (int u = 0; u < 16; u++)
                if (k0 + 16 * q + u < n_keys) mx = fmaxf(mx, v[u] * scale);
        }
    }
    VM_STAMP(9);
    if (WPQ > 1) {
        s_rowstat[hf][lr] = mx;
        pbar();
        mx = fmaxf(s_rowstat[0][lr], s_rowstat[1][lr]);
    }
    float sum = 0.f;
    for (int jb = 0; jb < g.nkb; jb++) {
        const int k0 = 128 * jb + KPT * hf;
#pragma unroll 1
        for (int q = 0; q < KPT / 16; q++) {
            if (k0 + 16 * q >= n_keys) break;
            float v[16];
            tmem_ld16(trow + 128 * jb + KPT * hf + 16 * q, v);
#pragma unroll
            for (int u = 0; u < 16; u++)
                if (k0 + 16 * q + u < n_keys) sum += ex2(fmaf(v[u], scale, -mx));
        }
    }
    if (WPQ > 1) {
        pbar();  // both halves have read the max
        s_rowstat[hf][lr] = sum;
        pbar();
        sum = s_rowstat[0][lr] + s_rowstat[1][lr];
    }
    const float inv = 1.0f / sum;
    VM_STAMP(4);
    VM_STAMP(10);
    // ---- per key block: P_j -> shared memory (SW128 K-major, chunk hf = keys [64 hf, 64 hf + 64)).
    //      V_j's chunks are loaded one block ahead (they only need ring slots), so each P.V MMA
    //      finds its operands resident as soon as P_j is written.
    const int vr = g.c0 + ar;  // value channel row of V^T loaded by this thread
    auto issue_v = [&](int jb) {
        const int nch = (attn_nb(n_keys, jb) + 63) / 64;
        if (tv) {
            if (tid == 0)
                for (int c = 0; c < nch; c++) {
                    const uint32_t sq = ps.it + c;
                    const int s = sq % STAGES;
                    if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                    expect_tx(s_bar + s, (uint32_t)(BK * DVS * 2));
                    tma2d(sbase + s * STAGE + A_BYTES, tv, 128 * jb + 64 * c, g.c0, s_bar + s);
                }
            ps.it += nch;
        } else {
            for (int c = 0; c < nch; c++) {
                const uint32_t sq = ps.it++;
                const int s = sq % STAGES;
                if (sq >= STAGES) mbar_wait((s_bar + STAGES) + s, ((sq / STAGES) & 1) ^ 1);
                const uint32_t sb = sbase + s * STAGE + A_BYTES;
                const int kv0 = 128 * jb + 64 * c;
                if (ar < DVS) {
                    const char* vs = vb + ((long long)vr * a.vt.ld + kv0) * 2;
#pragma unroll
                    for (int u = j0; u < j0 + CPT; u++) {
                        const bool ok = vr < a.dv && kv0 + 8 * u < n_keys;
                        cp_async16(sb + sw128_off(ar, u), ok ? (const void*)(vs + 16 * u) : (const void*)vb, ok);
                    }
                }
                cp_async_arrive_inc(s_bar + s);
                pbar();
                if (tid == 0) mbar_arrive(s_bar + s);
            }
        }
    };
    issue_v(0);
    for (int jb = 0; jb < g.nkb; jb++) {
        if (ps.pb > 0) mbar_wait_backoff((s_bar + 2 * STAGES + 3), (ps.pb - 1) & 1, 32);  // previous P.V MMAs done with the tile
        tc_fence_after();
        const int k0 = 128 * jb + KPT * hf;
#pragma unroll 1
        for (int q = 0; q < KPT / 16; q++) {
            unsigned char* pt = (vm_ring() + STAGES * STAGE + RES_BYTES) + ((KPT * hf + 16 * q) / 64) * (BM * 128);
            const int unit = ((16 * q) % 64) / 8;  // 16-byte unit of the 64-key SW128 chunk
            float v[16];
            if (k0 + 16 * q < n_keys) tmem_ld16(trow + 128 * jb + KPT * hf + 16 * q, v);
            uint4 pk[2];
            __nv_bfloat162* h = (__nv_bfloat162*)pk;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int kk = k0 + 16 * q + 2 * u;
                const float p0 = kk < n_keys ? ex2(fmaf(v[2 * u], scale, -mx)) * inv : 0.f;
                const float p1 = kk + 1 < n_keys ? ex2(fmaf(v[2 * u + 1], scale, -mx)) * inv : 0.f;
                h[u] = __floats2bfloat162_rn(p0, p1);
            }
            *(uint4*)(pt + sw128_off(lr, unit)) = pk[0];
            *(uint4*)(pt + sw128_off(lr, unit + 1)) = pk[1];
        }
        fence_async_smem();  // generic-proxy P writes -> tensor-core reads
        tc_fence_before();
        mbar_arrive((s_bar + 2 * STAGES + 2));
        ps.pb++;
        if (jb == 0) VM_STAMP(11);
        if (jb == g.nkb - 1) VM_STAMP(12);
        if (jb + 1 < g.nkb) issue_v(jb + 1);
    }
    // ---- epilogue: O slice (TMEM) -> staging -> + residual -> bf16 rows
    mbar_wait_backoff((s_bar + 2 * STAGES), ps.items & 1);
    ps.items++;
    tc_fence_after();
    VM_STAMP(5);
    constexpr int PLD = DVS + 4, hc = DVS / WPQ;
    float* stage = (float*)vm_ring();
    {
        const uint32_t taddr = trow + g.o_col + hf * hc;
        float* dst = stage + lr * PLD + hf * hc;
#pragma unroll 1
        for (int q = 0; q < hc / 16; q++) {
            float v[16];
            tmem_ld16(taddr + 16 * q, v);
#pragma unroll
            for (int w = 0; w < 4; w++)
                *(float4*)(dst + 16 * q + 4 * w) = make_float4(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]);
        }
        tc_fence_before();
    }
    if (staged) cp_wait<0>();
    pbar();
    const EpiCtx e = make_epi(s_ea, t);
    const int nrows = min(BM, a.m - g.m0);
    if (!e.pre && a.out.dtype == FIS_BF16 && (a.out.ld % 8) == 0 && (((uintptr_t)e.d) & 15) == 0 &&
        (staged || !e.res)) {
        fast_epilogue<DVS, FIS_EPI_NONE>(s_ea, e, sh, ge, stage, nullptr, 0, 1, 0, nrows, staged, tid);
    } else {
        for (int idx = tid; idx < nrows * (DVS / 8); idx += PRODUCERS) {
            const int row = idx / (DVS / 8), cb = (idx % (DVS / 8)) * 8;
            if (g.c0 + cb >= a.dv) continue;
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = stage[row * PLD + cb + u];
            EpiIn in;
            epilogue8_load(s_ea, e, g.m0 + row, g.c0 + cb, in, nullptr);
            epilogue8(s_ea, e, vm_tab(), g.m0 + row, cb, g.c0, v, in);
        }
    }
    VM_STAMP(6);
    signal_done(va, j, tid);
    VM_STAMP(7);
    if (va.trace_items && j == va.trace_op && tid == 0) va.trace_items[16 * i + 15] = clock64();
}

// ---------------------------------------------------------------------------------- SIMT ops
FIS_DEV float gather_a_simt(const fis_gemm_args& a, const char* f0, const char* c0p, const char* f1, const char* c1p,
                            const char* abase, int k, int p, int oy, int ox) {
    if (a.a_mode == FIS_A_ROWS) return load_elem(abase, a.a.dtype, (long long)p * a.a.ld + k);
    const int cin = a.src[0].c + (a.nsrc > 1 ? a.src[1].c : 0);
    const int tap = k / cin;
    int c = k - tap * cin;
    const int y = oy + tap / 3 - 1, x = ox + tap % 3 - 1;
    if (y < 0 || x < 0 || y >= a.out_h || x >= a.out_w) return 0.f;
    const bool second = c >= a.src[0].c;
    const fis_src& s = second ? a.src[1] : a.src[0];
    if (second) c -= a.src[0].c;
    const int sy = s.up ? (y >> 1) : y, sx = s.up ? (x >> 1) : x;
    return src_value(s, second ? f1 : f0, second ? c1p : c0p, sy * s.w + sx, c);
}

// Implicit 3x3 conv with 16-byte input pixels (the stem: 4 fp32 latent channels, unet.py:434):
// thread = (output pixel, 32-column half); its 9 taps are read once as float4 rows with
// select-on-read, the 64 x 36 weight tile sits in shared memory.  Same summation order as the
// SIMT tile (k ascending, fmaf), then the fis::epilogue_store operations.
__device__ __noinline__ bool stem_item(const fis_gemm_args& a, unsigned char* scratch, int item, int tiles_n, int tid) {
    const fis_src& sr = a.src[0];
    if (a.a_mode != FIS_A_CONV3X3 || a.nsrc != 1 || sr.c != 4 || sr.fresh.dtype != FIS_F32 || sr.up ||
        (sr.index && sr.cache.dtype != FIS_F32) || a.k != 36 || PRODUCERS != 128)
        return false;
    const int t = s_step;
    const int n0 = (item % tiles_n) * SBN, m0 = (item / tiles_n) * SBM;
    float* Ws = (float*)scratch;  // [SBN][37]
    const char* bbase = ref_base(a.b, t);
    for (int e = tid; e < SBN * 36; e += PRODUCERS) {
        const int n = e / 36, k = e % 36;
        Ws[n * 37 + k] = n0 + n < a.n ? load_elem(bbase, a.b.dtype, (long long)(n0 + n) * a.b.ld + k) : 0.f;
    }
    const char* fr = ref_base(sr.fresh, t);
    const char* ca = sr.index ? ref_base(sr.cache, t) : nullptr;
    const int lr = tid % SBM, half = tid / SBM;
    const int r = m0 + lr;
    float x[36];
    if (r < a.m) {
        const int p = a.rows ? __ldg(a.rows + r) : r;
        const int oy = p / a.out_w, ox = p - oy * a.out_w;
#pragma unroll
        for (int tap = 0; tap < 9; tap++) {
            const int y = oy + tap / 3 - 1, xx = ox + tap % 3 - 1;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (y >= 0 && xx >= 0 && y < a.out_h && xx < a.out_w) {
                const RowPtr rp = src_row(sr, fr, ca, y * sr.w + xx);
                v = FIS_LD_F4(rp.p);
            }
            x[4 * tap] = v.x; x[4 * tap + 1] = v.y; x[4 * tap + 2] = v.z; x[4 * tap + 3] = v.w;
        }
    }
    pbar();
    if (r >= a.m) return true;
    const EpiCtx e = make_epi(a, t);
    for (int cc = 0; cc < SBN / 2; cc++) {
        const int nl = half * (SBN / 2) + cc, n = n0 + nl;
        if (n >= a.n) break;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 36; k++) acc = fmaf(x[k], Ws[nl * 37 + k], acc);
        epilogue_store(a, e, r, n, acc);
    }
    return true;
}

__device__ __noinline__ void gemm_simt_item(const fis_gemm_args& a, unsigned char* scratch, int item, int tiles_n, int tid) {
    float (*As)[SBM + 4] = (float (*)[SBM + 4])scratch;
    float (*Bs)[SBN + 4] = (float (*)[SBN + 4])(scratch + SBK * (SBM + 4) * 4);
    int* rowp = (int*)(scratch + 2 * SBK * (SBM + 4) * 4);
    int* rowy = rowp + SBM;
    int* rowx = rowy + SBM;
    const int t = s_step;
    const int n0 = (item % tiles_n) * SBN, m0 = (item / tiles_n) * SBM;
    const char* abase = a.a.ptr ? ref_base(a.a, t) : nullptr;
    const char* f0 = a.nsrc > 0 && a.src[0].fresh.ptr ? ref_base(a.src[0].fresh, t) : nullptr;
    const char* c0p = a.nsrc > 0 && a.src[0].cache.ptr ? ref_base(a.src[0].cache, t) : nullptr;
    const char* f1 = a.nsrc > 1 && a.src[1].fresh.ptr ? ref_base(a.src[1].fresh, t) : nullptr;
    const char* c1p = a.nsrc > 1 && a.src[1].cache.ptr ? ref_base(a.src[1].cache, t) : nullptr;
    const char* bbase = ref_base(a.b, t);
    if (tid < SBM) {
        const int r = m0 + tid;
        const int p = r < a.m ? (a.rows ? __ldg(a.rows + r) : r) : 0;
        rowp[tid] = p;
        rowy[tid] = p / max(1, a.out_w);
        rowx[tid] = p - rowy[tid] * max(1, a.out_w);
    }
    pbar();
    constexpr int TY = PRODUCERS / 16, RPT = SBM / TY;  // thread grid 16 x TY, RPT rows x 4 columns each
    const int tx = tid % 16, ty = tid / 16;
    float acc[RPT][4];
#pragma unroll
    for (int i = 0; i < RPT; i++)
#pragma unroll
        for (int jj = 0; jj < 4; jj++) acc[i][jj] = 0.f;
    const int ktiles = (a.k + SBK - 1) / SBK;
    for (int kt = 0; kt < ktiles; kt++) {
        // the (row, k) elements of this pass: 32 A + 32 B gathers per thread, all independent
#pragma unroll 4
        for (int e = tid; e < SBM * SBK; e += PRODUCERS) {
            const int row = e / SBK, lk = e % SBK;
            const int k = kt * SBK + lk;
            const int r = m0 + row;
            float v = 0.f;
            if (r < a.m && k < a.k) v = gather_a_simt(a, f0, c0p, f1, c1p, abase, k, rowp[row], rowy[row], rowx[row]);
            As[lk][row] = v;
            const int n = n0 + row;
            float bv = 0.f;
            if (n < a.n && k < a.k) bv = load_elem(bbase, a.b.dtype, (long long)n * a.b.ld + k);
            Bs[lk][row] = bv;
        }
        pbar();
#pragma unroll
        for (int kk = 0; kk < SBK; kk++) {
            float av[RPT], bv[4];
#pragma unroll
            for (int i = 0; i < RPT; i++) av[i] = As[kk][ty * RPT + i];
#pragma unroll
            for (int jj = 0; jj < 4; jj++) bv[jj] = Bs[kk][tx * 4 + jj];
#pragma unroll
            for (int i = 0; i < RPT; i++)
#pragma unroll
                for (int jj = 0; jj < 4; jj++) acc[i][jj] = fmaf(av[i], bv[jj], acc[i][jj]);
        }
        pbar();
    }
    const EpiCtx e = make_epi(a, t);
    if (a.epi == FIS_EPI_NONE && !e.res && a.n_split == 0 && !a.d_trans && !a.d_rows) {
        // bias / time-bias columns read once (all loads in flight), then plain stores
        float bia[4], b2v[4];
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
            const int n = n0 + tx * 4 + jj;
            bia[jj] = n < a.n && a.bias ? __ldg(a.bias + n) : 0.f;
            b2v[jj] = n < a.n && e.bias2 ? load_elem(e.bias2, a.bias2.dtype, n) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < RPT; i++) {
            const int r = m0 + ty * RPT + i;
            if (r >= a.m) continue;
#pragma unroll
            for (int jj = 0; jj < 4; jj++) {
                const int n = n0 + tx * 4 + jj;
                if (n >= a.n) continue;
                float v = acc[i][jj] * a.alpha;  // same operation order as epilogue_store
                if (a.bias) v = __fadd_rn(v, bia[jj]);
                if (e.pre) store_elem(e.pre, a.pre.dtype, (long long)r * a.pre.ld + n, v);
                if (e.bias2) v = __fadd_rn(v, b2v[jj]);
                store_elem(e.d, a.d.dtype, (long long)r * a.d.ld + n, v);
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        const int r = m0 + ty * RPT + i;
        if (r >= a.m) continue;
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
            const int n = n0 + tx * 4 + jj;
            if (n < a.n) epilogue_store(a, e, r, n, acc[i][jj]);
        }
    }
}

// softmax rows [item*8, item*8+8): one warp per row (tensors.py:183-192, unet.py:555-566)
__device__ __noinline__ void softmax_item(const fis_softmax_args& a, int item, int tid) {
    const int t = s_step;
    const int row = item * SOFTMAX_ROWS + (tid >> 5);
    const int lane = tid & 31;
    if (row >= a.rows) return;
    char* pb = ref_base(a.p, t);
    char* mb = a.map.ptr ? ref_base(a.map, t) : nullptr;
    const float* cached = a.cached.ptr ? (const float*)ref_base(a.cached, t) + (long long)row * a.cached.ld : nullptr;
    const long long prow = (long long)row * a.p.ld;
    if (a.verbatim) {
        for (int jj = lane; jj < a.cols; jj += 32) {
            const float v = cached[jj];
            store_elem(pb, a.p.dtype, prow + jj, v);
            if (mb) ((float*)mb)[(long long)row * a.map.ld + jj] = v;
        }
    } else if (a.npairs == 0 && a.cols <= 32 * 16) {
        // one pass: the row lives in registers (<= 16 values per lane), all loads in flight at once
        const float* s = (const float*)ref_base(a.s, t) + (long long)row * a.s.ld;
        float x[16];
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const int jj = lane + 32 * k;
            x[k] = jj < a.cols ? __ldcg(s + jj) * a.scale : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < 16; k++) m = fmaxf(m, x[k]);
        m = warp_max(m);
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x[k] = lane + 32 * k < a.cols ? expf(x[k] - m) : 0.f;
            sum += x[k];
        }
        sum = warp_sum(sum);
        const float inv_sum = 1.0f / sum;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const int jj = lane + 32 * k;
            if (jj < a.cols) {
                const float v = x[k] * inv_sum;
                store_elem(pb, a.p.dtype, prow + jj, v);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + jj] = v;
            }
        }
    } else {
        const float* s = (const float*)ref_base(a.s, t) + (long long)row * a.s.ld;
        float m = -INFINITY;
        for (int jj = lane; jj < a.cols; jj += 32) m = fmaxf(m, __ldcg(s + jj) * a.scale);
        m = warp_max(m);
        float sum = 0.f;
        for (int jj = lane; jj < a.cols; jj += 32) sum += expf(__ldcg(s + jj) * a.scale - m);
        sum = warp_sum(sum);
        const float inv_sum = 1.0f / sum;
        if (a.npairs == 0) {
            for (int jj = lane; jj < a.cols; jj += 32) {
                const float v = expf(__ldcg(s + jj) * a.scale - m) * inv_sum;
                store_elem(pb, a.p.dtype, prow + jj, v);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + jj] = v;
            }
        } else {
            float rs = 0.f;
            for (int jj = lane; jj < a.cols; jj += 32) {
                float v = expf(__ldcg(s + jj) * a.scale - m) * inv_sum;
                for (int i = 0; i < a.npairs; i++)
                    if (__ldg(a.pair_new + i) == jj) v = cached[__ldg(a.pair_old + i)];
                rs += v;
            }
            rs = warp_sum(rs);
            for (int jj = lane; jj < a.cols; jj += 32) {
                float v = expf(__ldcg(s + jj) * a.scale - m) * inv_sum;
                for (int i = 0; i < a.npairs; i++)
                    if (__ldg(a.pair_new + i) == jj) v = cached[__ldg(a.pair_old + i)];
                const float o = (float)((double)v / (double)rs);
                store_elem(pb, a.p.dtype, prow + jj, o);
                if (mb) ((float*)mb)[(long long)row * a.map.ld + jj] = o;
            }
        }
    }
    for (int jj = a.cols + lane; jj < a.pad_cols; jj += 32) store_elem(pb, a.p.dtype, prow + jj, 0.f);
}

// group-norm statistics of group `g` (tensors.py:129-146): two-pass f64, rounded to f32
__device__ __noinline__ void gn_stats_item(const fis_gn_stats_args& a, double* red, int g, int tid) {
    const int t = s_step;
    const int cpg = a.c / a.groups;
    const long long cnt = (long long)a.hw * cpg;
    const char* x = ref_base(a.x, t);
    double s = 0.0;
    for (int q = tid; q < a.hw; q += PRODUCERS) {
        const long long base = (long long)q * a.x.ld + g * cpg;
        for (int c = 0; c < cpg; c++) s += (double)load_elem(x, a.x.dtype, base + c);
    }
    red[tid] = s;
    pbar();
    for (int o = PRODUCERS / 2; o; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        pbar();
    }
    const double mean = red[0] / (double)cnt;
    pbar();
    double v = 0.0;
    for (int q = tid; q < a.hw; q += PRODUCERS) {
        const long long base = (long long)q * a.x.ld + g * cpg;
        for (int c = 0; c < cpg; c++) {
            const double d = (double)load_elem(x, a.x.dtype, base + c) - mean;
            v += d * d;
        }
    }
    red[tid] = v;
    pbar();
    for (int o = PRODUCERS / 2; o; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        pbar();
    }
    if (tid == 0) {
        ((float*)ref_base(a.mean, t))[g] = (float)mean;
        ((float*)ref_base(a.var, t))[g] = (float)(red[0] / (double)cnt);
    }
}

__device__ __noinline__ void gn_apply_item(const fis_gn_apply_args& a, int item, int tid) {
    const int t = s_step;
    const char* x = ref_base(a.x, t);
    const float* mean = (const float*)ref_base(a.mean, t);
    const float* var = (const float*)ref_base(a.var, t);
    char* yn = a.y_norm.ptr ? ref_base(a.y_norm, t) : nullptr;
    char* ys = a.y_silu.ptr ? ref_base(a.y_silu, t) : nullptr;
    const int cpg = a.c / a.groups;
    const int total = a.rows * a.c;
    const int e1 = min(total, (item + 1) * ELEMS_PER_ITEM);
    for (int e = item * ELEMS_PER_ITEM + tid; e < e1; e += PRODUCERS) {
        const int r = e / a.c, c = e - (e / a.c) * a.c;
        const int xr = a.x_rows ? __ldg(a.x_rows + r) : r;
        const int yr = a.y_rows ? __ldg(a.y_rows + r) : r;
        const int g = c / cpg;
        const double xv = (double)load_elem(x, a.x.dtype, (long long)xr * a.x.ld + c);
        const double y64 = (xv - (double)mean[g]) / sqrt((double)var[g] + (double)a.eps) * (double)a.gamma[c] +
                           (double)a.beta[c];
        const float y = (float)y64;
        if (yn) store_elem(yn, a.y_norm.dtype, (long long)yr * a.y_norm.ld + c, y);
        if (ys) {
            const double yd = (double)y;
            store_elem(ys, a.y_silu.dtype, (long long)yr * a.y_silu.ld + c, (float)(yd / (1.0 + exp(-yd))));
        }
    }
}

__device__ __noinline__ void pool_item(const fis_pool_args& a, int item, int tid) {
    const int t = s_step;
    const char* fr = a.src.fresh.ptr ? ref_base(a.src.fresh, t) : nullptr;
    const char* ca = a.src.cache.ptr ? ref_base(a.src.cache, t) : nullptr;
    char* out = ref_base(a.out, t);
    const int cw = a.src.w / 2;
    const int total = a.n * a.c;
    const int e1 = min(total, (item + 1) * ELEMS_PER_ITEM);
    const bool vec = a.src.fresh.dtype == FIS_BF16 && (!a.src.index || a.src.cache.dtype == FIS_BF16) &&
                     a.out.dtype == FIS_BF16 && (a.c % 8) == 0 && (a.src.fresh.ld % 8) == 0 &&
                     (!a.src.index || (a.src.cache.ld % 8) == 0) && (a.out.ld % 8) == 0 &&
                     ((((uintptr_t)fr) | ((uintptr_t)ca) | ((uintptr_t)out)) & 15) == 0;
    if (vec) {
        // 8 channels (16 bytes) per unit: the 4 source rows are selected once, read as one vector each
        for (int e = item * ELEMS_PER_ITEM + tid * 8; e < e1; e += PRODUCERS * 8) {
            const int i = e / a.c, c = e - (e / a.c) * a.c;
            const int P = a.rows ? __ldg(a.rows + i) : i;
            const int py = P / cw, px = P - (P / cw) * cw;
            const int q = (2 * py) * a.src.w + 2 * px;
            const int qs[4] = {q, q + 1, q + a.src.w, q + a.src.w + 1};
            uint4 u[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const RowPtr rp = src_row(a.src, fr, ca, qs[k]);
                u[k] = FIS_LD_U4((const __nv_bfloat16*)rp.p + c);
            }
            uint4 o;
            __nv_bfloat162* oh = (__nv_bfloat162*)&o;
#pragma unroll
            for (int h = 0; h < 4; h++) {
                const float2 a0 = __bfloat1622float2(((const __nv_bfloat162*)&u[0])[h]);
                const float2 a1 = __bfloat1622float2(((const __nv_bfloat162*)&u[1])[h]);
                const float2 a2 = __bfloat1622float2(((const __nv_bfloat162*)&u[2])[h]);
                const float2 a3 = __bfloat1622float2(((const __nv_bfloat162*)&u[3])[h]);
                oh[h] = __floats2bfloat162_rn(__fmul_rn(__fadd_rn(__fadd_rn(a0.x, a1.x), __fadd_rn(a2.x, a3.x)), 0.25f),
                                              __fmul_rn(__fadd_rn(__fadd_rn(a0.y, a1.y), __fadd_rn(a2.y, a3.y)), 0.25f));
            }
            *(uint4*)((__nv_bfloat16*)out + (long long)i * a.out.ld + c) = o;
        }
        return;
    }
    for (int e = item * ELEMS_PER_ITEM + tid; e < e1; e += PRODUCERS) {
        const int i = e / a.c, c = e - (e / a.c) * a.c;
        const int P = a.rows ? __ldg(a.rows + i) : i;
        const int py = P / cw, px = P - (P / cw) * cw;
        const int q = (2 * py) * a.src.w + 2 * px;
        const float v00 = src_value(a.src, fr, ca, q, c), v01 = src_value(a.src, fr, ca, q + 1, c);
        const float v10 = src_value(a.src, fr, ca, q + a.src.w, c), v11 = src_value(a.src, fr, ca, q + a.src.w + 1, c);
        const float s = __fadd_rn(__fadd_rn(v00, v01), __fadd_rn(v10, v11));
        store_elem(out, a.out.dtype, (long long)i * a.out.ld + c, __fmul_rn(s, 0.25f));
    }
}

// Group norm of one group (item = group): two-pass f64 statistics over the full map (rounded to
// f32, tensors.py:129-146), written to mean/var, then the group's channels normalised with them
// (+ SiLU) in fp32 (bf16 step VM).  Fuses group_norm's reduction and normalize_with_group_stats.
__device__ __noinline__ void gn_item(const fis_gn_apply_args& a, double* red, int g, int tid) {
    const int t = s_step;
    const char* x = ref_base(a.x, t);
    const int cpg = a.c / a.groups;
    const int hw = a.rows;
    const long long cnt = (long long)hw * cpg;
    const int c0 = g * cpg;
    auto reduce = [&](double v) -> double {
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0) red[tid >> 5] = v;
        pbar();
        double r = 0.0;
        for (int w = 0; w < PRODUCERS / 32; w++) r += red[w];
        pbar();
        return r;
    };
    char* yn = a.y_norm.ptr ? ref_base(a.y_norm, t) : nullptr;
    char* ys = a.y_silu.ptr ? ref_base(a.y_silu, t) : nullptr;
    const int vpr = cpg / 8;  // 16-byte vectors of the group per pixel
    constexpr int MAXV = 12;  // group data held in registers: <= MAXV * PRODUCERS vectors
    const bool vec = a.x.dtype == FIS_BF16 && (cpg % 8) == 0 && (a.x.ld % 8) == 0 && (c0 % 8) == 0 &&
                     hw * vpr <= MAXV * PRODUCERS && (!yn || a.y_norm.dtype == FIS_BF16) &&
                     (!ys || a.y_silu.dtype == FIS_BF16) && (((uintptr_t)x) & 15) == 0;
    if (vec) {
        // one vectorised read of the group into registers, f64 two-pass statistics from them
        uint4 u[MAXV];
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < MAXV; k++) {
            const int e = tid + k * PRODUCERS;
            if (e < hw * vpr) {
                const int q = e / vpr, c = c0 + 8 * (e % vpr);
                u[k] = FIS_LD_U4((const __nv_bfloat16*)x + (long long)q * a.x.ld + c);
                const __nv_bfloat162* h = (const __nv_bfloat162*)&u[k];
#pragma unroll
                for (int w = 0; w < 4; w++) {
                    const float2 f = __bfloat1622float2(h[w]);
                    s += (double)f.x;
                    s += (double)f.y;
                }
            }
        }
        const double mean = reduce(s) / (double)cnt;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < MAXV; k++) {
            const int e = tid + k * PRODUCERS;
            if (e < hw * vpr) {
                const __nv_bfloat162* h = (const __nv_bfloat162*)&u[k];
#pragma unroll
                for (int w = 0; w < 4; w++) {
                    const float2 f = __bfloat1622float2(h[w]);
                    const double d0 = (double)f.x - mean, d1 = (double)f.y - mean;
                    v += d0 * d0;
                    v += d1 * d1;
                }
            }
        }
        const double var = reduce(v) / (double)cnt;
        const float mean_f = (float)mean, var_f = (float)var;
        if (tid == 0) {
            ((float*)ref_base(a.mean, t))[g] = mean_f;
            ((float*)ref_base(a.var, t))[g] = var_f;
        }
        const float rstd = (float)(1.0 / sqrt((double)var_f + (double)a.eps));
#pragma unroll
        for (int k = 0; k < MAXV; k++) {
            const int e = tid + k * PRODUCERS;
            if (e < hw * vpr) {
                const int q = e / vpr, c = c0 + 8 * (e % vpr);
                const __nv_bfloat162* h = (const __nv_bfloat162*)&u[k];
                uint4 on, os;
                __nv_bfloat162* hn = (__nv_bfloat162*)&on;
                __nv_bfloat162* hs = (__nv_bfloat162*)&os;
#pragma unroll
                for (int w = 0; w < 4; w++) {
                    const float2 f = __bfloat1622float2(h[w]);
                    const float y0 = fmaf((f.x - mean_f) * rstd, __ldg(a.gamma + c + 2 * w), __ldg(a.beta + c + 2 * w));
                    const float y1 = fmaf((f.y - mean_f) * rstd, __ldg(a.gamma + c + 2 * w + 1), __ldg(a.beta + c + 2 * w + 1));
                    hn[w] = __floats2bfloat162_rn(y0, y1);
                    hs[w] = __floats2bfloat162_rn(__fdividef(y0, 1.0f + __expf(-y0)), __fdividef(y1, 1.0f + __expf(-y1)));
                }
                if (yn) *(uint4*)((__nv_bfloat16*)yn + (long long)q * a.y_norm.ld + c) = on;
                if (ys) *(uint4*)((__nv_bfloat16*)ys + (long long)q * a.y_silu.ld + c) = os;
            }
        }
        return;
    }
    double s = 0.0;
    for (int e = tid; e < hw * cpg; e += PRODUCERS) {
        const int q = e / cpg, c = c0 + (e - (e / cpg) * cpg);
        s += (double)load_elem(x, a.x.dtype, (long long)q * a.x.ld + c);
    }
    const double mean = reduce(s) / (double)cnt;
    double v = 0.0;
    for (int e = tid; e < hw * cpg; e += PRODUCERS) {
        const int q = e / cpg, c = c0 + (e - (e / cpg) * cpg);
        const double d = (double)load_elem(x, a.x.dtype, (long long)q * a.x.ld + c) - mean;
        v += d * d;
    }
    const double var = reduce(v) / (double)cnt;
    const float mean_f = (float)mean, var_f = (float)var;
    if (tid == 0) {
        ((float*)ref_base(a.mean, t))[g] = mean_f;
        ((float*)ref_base(a.var, t))[g] = var_f;
    }
    const float rstd = (float)(1.0 / sqrt((double)var_f + (double)a.eps));
    for (int e = tid; e < hw * cpg; e += PRODUCERS) {
        const int q = e / cpg, c = c0 + (e - (e / cpg) * cpg);
        const float xv = load_elem(x, a.x.dtype, (long long)q * a.x.ld + c);
        const float y = fmaf((xv - mean_f) * rstd, __ldg(a.gamma + c), __ldg(a.beta + c));
        if (yn) store_elem(yn, a.y_norm.dtype, (long long)q * a.y_norm.ld + c, y);
        if (ys) store_elem(ys, a.y_silu.dtype, (long long)q * a.y_silu.ld + c, __fdividef(y, 1.0f + __expf(-y)));
    }
}

__device__ __noinline__ void materialize_item(const fis_materialize_args& a, int item, int tid) {
    const int t = s_step;
    const char* fr = a.src.fresh.ptr ? ref_base(a.src.fresh, t) : nullptr;
    const char* ca = a.src.cache.ptr ? ref_base(a.src.cache, t) : nullptr;
    char* out = ref_base(a.out, t);
    const int total = a.src.h * a.src.w * a.c;
    const int e1 = min(total, (item + 1) * ELEMS_PER_ITEM);
    for (int e = item * ELEMS_PER_ITEM + tid; e < e1; e += PRODUCERS) {
        const int q = e / a.c, c = e - (e / a.c) * a.c;
        store_elem(out, a.out.dtype, (long long)q * a.out.ld + c, src_value(a.src, fr, ca, q, c));
    }
}

FIS_DEV void producer_role(const fis_vm_args& va, const Shared& sh, uint32_t tmem, int tid) {
    const int G = gridDim.x, cta = blockIdx.x;
    ProdState ps{0, 0, 0, 0, 0};
    for (int j = 0; j < va.n_ops; j++) {
        const fis_vm_op* gop = va.ops + j;
        const int n_items = gop->n_items;
        int i = (cta - gop->cta0 + G) % G;
        if (i >= n_items) continue;
        // stage the op record in shared memory (previous op's readers are past their last barrier)
        pbar();
        {
            static_assert(sizeof(fis_vm_op) % 8 == 0, "fis_vm_op is copied as 8-byte words");
            const long long* src = (const long long*)gop;
            long long* dst = (long long*)(&s_op);
            for (int w = tid; w < (int)sizeof(fis_vm_op) / 8; w += PRODUCERS) dst[w] = __ldg(src + w);
        }
        pbar();
        const fis_vm_op& op = s_op;
        bool waited = false;
        for (; i < n_items; i += G) {
            switch (op.kind) {
                case FIS_VM_GEMM:
                    if (op.impl == 2) {
                        if (op.bn == 64) gemm_tc_item<64>(va, sh, j, i, ps, waited, tmem, tid);
                        else gemm_tc_item<128>(va, sh, j, i, ps, waited, tmem, tid);
                    } else {
                        VM_STAMP(0);
                        wait_dep(va, op, j, waited, tid);
                        VM_STAMP(2);
                        if (!stem_item(op.u.gemm, vm_ring(), i, op.tiles_n, tid))
                            gemm_simt_item(op.u.gemm, vm_ring(), i, op.tiles_n, tid);
                        VM_STAMP(6);
                        signal_done(va, j, tid);
                        VM_STAMP(7);
                    }
                    break;
                case FIS_VM_ATTN:
                    if (op.bn == 64) attn_item_run<64>(va, sh, j, i, ps, waited, tmem, tid);
                    else attn_item_run<128>(va, sh, j, i, ps, waited, tmem, tid);
                    break;
                case FIS_VM_SOFTMAX:
                    VM_STAMP(0);
                    wait_dep(va, op, j, waited, tid);
                    VM_STAMP(2);
                    softmax_item(op.u.softmax, i, tid);
                    VM_STAMP(6);
                    signal_done(va, j, tid);
                    VM_STAMP(7);
                    break;
                case FIS_VM_GN_STATS:
                    wait_dep(va, op, j, waited, tid);
                    gn_stats_item(op.u.gn_stats, (double*)vm_ring(), i, tid);
                    signal_done(va, j, tid);
                    break;
                case FIS_VM_GN:
                    VM_STAMP(0);
                    wait_dep(va, op, j, waited, tid);
                    VM_STAMP(2);
                    gn_item(op.u.gn_apply, (double*)vm_ring(), i, tid);
                    VM_STAMP(6);
                    signal_done(va, j, tid);
                    break;
                case FIS_VM_GN_APPLY:
                    wait_dep(va, op, j, waited, tid);
                    gn_apply_item(op.u.gn_apply, i, tid);
                    signal_done(va, j, tid);
                    break;
                case FIS_VM_POOL:
                    wait_dep(va, op, j, waited, tid);
                    pool_item(op.u.pool, i, tid);
                    signal_done(va, j, tid);
                    break;
                case FIS_VM_MATERIALIZE:
                    wait_dep(va, op, j, waited, tid);
                    materialize_item(op.u.materialize, i, tid);
                    signal_done(va, j, tid);
                    break;
                default:
                    break;
            }
        }
    }
}

__global__ void __launch_bounds__(THREADS, 1) vm_kernel(const fis_vm_args va) {
    const Shared sh = carve();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(s_bar + s, 1);  // thread 0's arrival (+ TMA bytes, + incrementing cp.async arrivals)
            mbar_init((s_bar + STAGES) + s, 1);
        }
        mbar_init((s_bar + 2 * STAGES), 1);
        mbar_init((s_bar + 2 * STAGES + 1), 1);
        mbar_init((s_bar + 2 * STAGES + 2), PRODUCERS);
        mbar_init((s_bar + 2 * STAGES + 3), 1);
        mbar_init((s_bar + 2 * STAGES + 4), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32((&s_tmem))),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *(&s_tmem);
    if (tid == 0) s_step = va.step ? *va.step : 0;
    __syncthreads();

    if (warp == MMA_WARP) mma_role(va, sh, tmem, lane);
    else if (tid < PRODUCERS) producer_role(va, sh, tmem, tid);

    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    // the last CTA to leave resets the per-op completion counters for the next launch
    if (tid == 0) {
        __threadfence();
        const int old = atomicAdd(va.sync, 1);
        if (old == (int)gridDim.x - 1) {
            for (int j = 1; j < va.n_sync; j++) va.sync[j] = 0;
            __threadfence();
            va.sync[0] = 0;
        }
    }
}

}  // namespace vm
}  // namespace fis

int fis_gemm_tc_supported(const fis_gemm_args* a);

#include "fis_tma.cuh"

static int vm_sm_count() {
    static int n = 0;
    if (n <= 0) n = fis_device_sm_count();
    return n > 0 ? n : 148;
}

extern "C" int fis_vm_op_size(void) { return (int)sizeof(fis_vm_op); }

// Value-slice width of a VM attention op (64 or 128 columns dividing dv) such that the key
// blocks (16-column rounded) and the O slice fit the 512 TMEM columns; 0 = not supported.
extern "C" int fis_vm_attn_slice(int m, int n_keys, int d, int dv) {
    if (!VM_FUSED_ATTN) return 0;
    if (m < 0 || n_keys < 1 || d % 64 || dv <= 0) return 0;
    const int s_cols = 128 * ((n_keys - 1) / 128) + ((n_keys - 128 * ((n_keys - 1) / 128) + 15) & ~15);
    for (int w = 128; w >= 64; w -= 64)
        if (dv % w == 0 && s_cols + w <= fis::vm::TMEM_COLS) return w;
    return 0;
}

// 3-D bf16 tensor map of a dense conv source [h][w][c] (pixel stride ld), box {64, w, 128 / w}:
// one tap of a 128-pixel output tile.
static bool encode_conv(void* out128, const fis_src& s, int out_h, int out_w) {
    if (s.index || s.up || s.fresh.step_stride || s.fresh.dtype != FIS_BF16 || !s.fresh.ptr) return false;
    if (s.h != out_h || s.w != out_w || out_w > 128 || 128 % out_w || (s.c % 64)) return false;
    const void* base = s.fresh.ptr;
    const long long ld = s.fresh.ld;
    if ((((uintptr_t)base) & 15) || ((ld * 2) % 16) || ld < s.c) return false;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)s.c, (cuuint64_t)s.w, (cuuint64_t)s.h};
    cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(ld * 2 * s.w)};
    cuuint32_t box[3] = {64u, (cuuint32_t)out_w, (cuuint32_t)(128 / out_w)};
    cuuint32_t es[3] = {1u, 1u, 1u};
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                                              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out128, &m, 128);
    return true;
}

extern "C" int fis_vm_plan(fis_vm_op* ops, int n, int n_ctas, long long* ws_floats, int* sync_ints) {
    int nt = 0;
    return fis_vm_plan_tma(ops, n, n_ctas, ws_floats, sync_ints, nullptr, 0, &nt);
}

extern "C" int fis_vm_plan_tma(fis_vm_op* ops, int n, int n_ctas, long long* ws_floats, int* sync_ints, void* tmaps,
                               int cap, int* n_tmaps) {
    int nt = 0;
    // FIS_VM_TMA_MASK (debug): 1 B operands, 2 row-major A, 4 dense-conv A, 8 attention (default all)
    const char* mask_env = getenv("FIS_VM_TMA_MASK");
    const int tma_mask = mask_env ? atoi(mask_env) : 15;
    using namespace fis::vm;
    const int G = n_ctas > 0 ? n_ctas : vm_sm_count();
    long long ws = 0;
    int sync_next = 1 + n;
    int cta = 0, last = -1;
    for (int j = 0; j < n; j++) {
        fis_vm_op& op = ops[j];
        op.impl = 0; op.bn = 0; op.tiles_n = 0; op.tiles_m = 0; op.splits = 1; op.sync_base = 0;
        op.tmap_a = -1; op.tmap_b = -1; op.tmap_a2 = -1; op.pad_ = 0;
        switch (op.kind) {
            case FIS_VM_GEMM: {
                const fis_gemm_args& a = op.u.gemm;
                if (a.m < 0 || a.n <= 0 || a.k <= 0) return FIS_ERR_SHAPE;
                if (a.a_mode == FIS_A_CONV3X3) {
                    if (a.nsrc < 1 || a.nsrc > 2) return FIS_ERR_SHAPE;
                    const int cin = a.src[0].c + (a.nsrc > 1 ? a.src[1].c : 0);
                    if (a.k != 9 * cin) return FIS_ERR_SHAPE;
                    for (int i = 0; i < a.nsrc; i++)
                        if (a.src[i].index && !a.src[i].cache.ptr) return FIS_ERR_CACHE_MISS;
                }
                if (a.epi == FIS_EPI_GN_SILU && (a.groups <= 0 || a.n % a.groups || !a.gn_mean.ptr || !a.gn_var.ptr))
                    return FIS_ERR_SHAPE;
                if (a.epi == FIS_EPI_STEP && a.res.ptr) return FIS_ERR_UNSUPPORTED;  // one epilogue read per item
                const bool tc = a.impl != 1 && fis_gemm_tc_supported(&a);
                if (tc) {
                    op.impl = 2;
                    const int kb = (a.k + BK - 1) / BK;
                    // 64-column tiles when that gives more tiles for a short K (no split-K to pay)
                    const int t128 = ((a.n + 127) / 128) * ((a.m + BM - 1) / BM);
                    op.bn = (a.n <= 64 || (kb < VM_MIN_SPLIT_KB && t128 * 2 <= G)) ? 64 : 128;
                    op.tiles_n = (a.n + op.bn - 1) / op.bn;
                    op.tiles_m = (a.m + BM - 1) / BM;
                    const int tiles = op.tiles_n * op.tiles_m;
                    // split-K: every split CTA of a tile must be co-resident (they meet at a tile
                    // counter), so tiles * S <= G.  A split costs a partial exchange (~4 us), so
                    // only K ranges long enough to stream for longer than that are split.
                    int S = a.splits > 0 ? a.splits : G / (tiles > 0 ? tiles : 1);
                    if (a.splits <= 0 && S > kb / (VM_MIN_SPLIT_KB / 2)) S = kb / (VM_MIN_SPLIT_KB / 2);
                    if (S > G / (tiles > 0 ? tiles : 1)) S = G / (tiles > 0 ? tiles : 1);
                    if (S > 32) S = 32;
                    if (S < 1) S = 1;
                    const int per = (kb + S - 1) / S;
                    S = (kb + per - 1) / per;
                    op.splits = S;
                    op.n_items = tiles * S;
                    op.n_done = tiles * S;
                    // TMA for B (weights, K/V operands) and for plain row-major A
                    if (tmaps && (tma_mask & 1) && nt < cap && a.b.step_stride == 0 &&
                        encode_2d((char*)tmaps + 128 * nt, a.b.ptr, a.n, a.k, a.b.ld, op.bn))
                        op.tmap_b = nt++;
                    if (tmaps && (tma_mask & 2) && nt < cap && a.a_mode == FIS_A_ROWS && !a.rows && a.a.step_stride == 0 &&
                        a.a.dtype == FIS_BF16 && encode_2d((char*)tmaps + 128 * nt, a.a.ptr, a.m, a.k, a.a.ld, BM))
                        op.tmap_a = nt++;
                    if (tmaps && (tma_mask & 4) && a.a_mode == FIS_A_CONV3X3 && !a.rows) {  // dense conv: per-tap boxes
                        if (nt < cap && encode_conv((char*)tmaps + 128 * nt, a.src[0], a.out_h, a.out_w)) op.tmap_a = nt++;
                        if (a.nsrc > 1 && nt < cap && encode_conv((char*)tmaps + 128 * nt, a.src[1], a.out_h, a.out_w))
                            op.tmap_a2 = nt++;
                    }
                    if (S > 1) {
                        op.sync_base = sync_next;
                        sync_next += tiles;
                        const long long need = (long long)tiles * S * BM * op.bn;
                        if (need > ws) ws = need;
                    }
                } else {
                    op.impl = 1;
                    op.tiles_n = (a.n + SBN - 1) / SBN;
                    op.tiles_m = (a.m + SBM - 1) / SBM;
                    op.n_items = op.tiles_n * op.tiles_m;
                    op.n_done = op.n_items;
                }
                break;
            }
            case FIS_VM_SOFTMAX: {
                const fis_softmax_args& a = op.u.softmax;
                if (a.pad_cols < a.cols) return FIS_ERR_SHAPE;
                if ((a.verbatim || a.npairs) && !a.cached.ptr) return FIS_ERR_CACHE_MISS;
                op.n_items = (a.rows + SOFTMAX_ROWS - 1) / SOFTMAX_ROWS;
                break;
            }
            case FIS_VM_GN_STATS:
                if (op.u.gn_stats.groups <= 0 || op.u.gn_stats.c % op.u.gn_stats.groups) return FIS_ERR_SHAPE;
                op.n_items = op.u.gn_stats.groups;
                break;
            case FIS_VM_GN: {
                const fis_gn_apply_args& a = op.u.gn_apply;
                if (a.groups <= 0 || a.c % a.groups || a.x_rows || a.y_rows) return FIS_ERR_SHAPE;
                op.n_items = a.rows > 0 ? a.groups : 0;
                break;
            }
            case FIS_VM_GN_APPLY: {
                const fis_gn_apply_args& a = op.u.gn_apply;
                if (a.groups <= 0 || a.c % a.groups) return FIS_ERR_SHAPE;
                op.n_items = (int)(((long long)a.rows * a.c + ELEMS_PER_ITEM - 1) / ELEMS_PER_ITEM);
                break;
            }
            case FIS_VM_POOL:
                if (op.u.pool.src.index && !op.u.pool.src.cache.ptr) return FIS_ERR_CACHE_MISS;
                op.n_items = (int)(((long long)op.u.pool.n * op.u.pool.c + ELEMS_PER_ITEM - 1) / ELEMS_PER_ITEM);
                break;
            case FIS_VM_MATERIALIZE: {
                const fis_materialize_args& a = op.u.materialize;
                if (a.src.index && !a.src.cache.ptr) return FIS_ERR_CACHE_MISS;
                op.n_items = (int)(((long long)a.src.h * a.src.w * a.c + ELEMS_PER_ITEM - 1) / ELEMS_PER_ITEM);
                break;
            }
            case FIS_VM_ATTN: {
                const fis_attn_args& a = op.u.attn;
                const int dvs = fis_vm_attn_slice(a.m, a.n_keys, a.d, a.dv);
                if (!dvs || a.q.dtype != FIS_BF16 || a.k.dtype != FIS_BF16 || a.vt.dtype != FIS_BF16 ||
                    (a.q.ld % 8) || (a.k.ld % 8) || (a.vt.ld % 8))
                    return FIS_ERR_UNSUPPORTED;
                op.bn = dvs;
                op.tiles_n = a.dv / dvs;
                op.tiles_m = (a.m + BM - 1) / BM;
                op.n_items = a.m > 0 ? op.tiles_n * op.tiles_m : 0;
                if (tmaps && (tma_mask & 8) && a.q.step_stride == 0 && a.k.step_stride == 0 && a.vt.step_stride == 0 &&
                    nt + 3 <= cap) {
                    if (encode_2d((char*)tmaps + 128 * nt, a.q.ptr, a.m, a.d, a.q.ld, BM)) op.tmap_a = nt++;
                    if (encode_2d((char*)tmaps + 128 * nt, a.k.ptr, a.n_keys, a.d, a.k.ld, 128)) op.tmap_b = nt++;
                    if (encode_2d((char*)tmaps + 128 * nt, a.vt.ptr, a.dv, a.n_keys, a.vt.ld, dvs)) op.tmap_a2 = nt++;
                }
                break;
            }
            default:
                return FIS_ERR_UNSUPPORTED;
        }
        if (op.kind != FIS_VM_GEMM) op.n_done = op.n_items;
        op.dep = last;
        op.dep_target = last >= 0 ? ops[last].n_done : 0;
        op.cta0 = cta;
        cta = (int)((cta + (long long)op.n_items) % G);
        if (op.n_items > 0) last = j;
    }
    if (ws_floats) *ws_floats = ws;
    if (sync_ints) *sync_ints = sync_next;
    if (n_tmaps) *n_tmaps = nt;
    return FIS_OK;
}

extern "C" int fis_vm_run(const fis_vm_args* a, void* stream) {
    using namespace fis::vm;
    if (a->n_ops <= 0) return FIS_OK;
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(vm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
            return FIS_ERR_UNSUPPORTED;
        configured = true;
    }
    const int G = a->n_ctas > 0 ? a->n_ctas : vm_sm_count();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = (cudaStream_t)stream;
    // all CTAs must be co-resident (items wait on other CTAs): cooperative launch guarantees it
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, vm_kernel, *a) == cudaSuccess ? FIS_OK : FIS_ERR_LAUNCH;
}
