// Dual-scope attention core, TMA ring (attend_tokens, ops.cpp:209-241, applied per spatial
// position as in dual_scope_reference ops.cpp:318-336 and attention_parallel
// clip_parallel.cpp:311-334). The Q/K/V projections run before it as tcgen05 GEMMs; the core
// does only the banded + global token mixing, ~1.5% of the block's flops, bound by reading
// Q/K/V once and writing ctx once. launch_attention_core feeds narrow bf16 tiles
// (<= 32 distinct K/V frames per 32-query block: the 24-frame VideoCrafter2 clip, the
// headline) through this TMA ring and everything else through attention_cpasync.cu:
//
//   * work item = (spatial position p, block of 32 query frames); R = the distinct K/V
//     frames the block's queries touch (window band + sampled globals);
//   * persistent CTAs, warp-specialised: one producer warp issues TMA loads (4-D tensor maps
//     over the [frames][HW][3 x heads][d] Q/K/V buffer, 128-byte swizzle, 64-wide head-dim
//     chunks, zero-filled past the head dim) into one mbarrier FIFO ring per CTA: a block's
//     query rows are one box, its K/V frames a host-built program of one box per run of
//     consecutive frames (<= 32 rows) or one row gather per four isolated frames (instances
//     with a compile-time head dim add a copy warp that moves the query rows with cp.async
//     instead: the TMA engine's per-row cost bounds the feed, the LSU path runs beside it); four
//     consumer warps: S = Q K^T per head over the chunks, the reference's explicit token
//     softmax (window tokens then globals, duplicates kept, +bias on the flagged side) in
//     column form, ctx = P V chunk by chunk through per-warp staging to 16-byte stores;
//   * mma.sync m16n8k16 bf16 -> fp32 (tcgen05 needs M >= 64; a block has <= 32 queries, 24 at
//     the VideoCrafter2 clip);
//   * bf16 mode: Q/K/V and ctx are bf16; split mode (the fp32 engine mode): each is two bf16
//     planes hi = RN(x), lo = RN(x - hi) and every product runs as hi*hi + hi*lo + lo*hi (S
//     and PV), the same bf16x3 arithmetic as the fp32-mode GEMMs.
//
// The FIFO keeps a fixed prefetch distance across phases and items: V chunks load during the
// softmax, the next item's Q/K chunks during the PV phase.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn();
// widest K/V list (rows) the copy-warp TMA instances take for one-block clips
// (VINF_ATTN_CW_ROWS, diagnostics)
static const uint32_t g_cw_rows = [] {
    const char* e = getenv("VINF_ATTN_CW_ROWS");
    return e ? uint32_t(atoi(e)) : 64u;
}();
int g_attn_impl = []() {  // 0 = by configuration, 1 = TMA ring, 2 = cp.async ring (diagnostics)
    const char* e = getenv("VINF_ATTN_IMPL");
    if (!e) return 0;
    const std::string v(e);
    return v == "tma" ? 1 : v == "cpasync" ? 2 : 0;
}();

namespace {

constexpr int kDC = 64;  // head-dim chunk (one 128-byte swizzle row of bf16)
// CW consumer warps per CTA (4 in every instance) + one producer warp; derived tile constants:
#define VINF_ATTN_WARP_CONSTANTS(CW)                                                         \
    static constexpr int kConsumerWarps = CW;                                                  \
    static constexpr int kThreads = (kConsumerWarps + 1) * 32; /* + the producer warp */      \
    static constexpr int kWQ = kConsumerWarps / 2;             /* warps per 16-query m tile */ \
    static constexpr int kON = 8 / kWQ;  /* PV: n8 output tiles per warp in a 64-wide chunk */ \
    static constexpr uint32_t kOPitch = kON * 16 + 16; /* ctx staging row pitch, conflict-free */
constexpr uint32_t kQT = kQBlock * 128;  // one plane of a Q chunk (32 rows x 128 B)

struct AttnMaps {
    CUtensorMap box[2][kBoxKinds];  // [plane][kind]: boxes of kind + 1 frames x 64 head-dim elements
    CUtensorMap g4[2];              // [plane]: 2-D rows x 3C view, box {64, 1}, for row gathers
};

struct AttnArgs {
    uint32_t HW, C, heads, d, nch, nq, nqb, q_frame0, items, ns;
    uint32_t load_only;  // diagnostics: 1 = the feed alone (consumers only release stages), 3 = no loads
    uint32_t qfeed;      // D > 0 instances: 1 = Q rows (and residual chunks) by the copy warp (cp.async)
    const __nv_bfloat16* q;     // the Q/K/V buffer (and its lo plane) for the copy warp
    const __nv_bfloat16* q_lo;
    float scale, bias;
    __nv_bfloat16* ctx;
    int64_t ctx_lo;  // elements from ctx to its lo plane (split mode)
    FuseO fo;        // fo.y: the block output (O projection absorbed into V) instead of ctx
    uint32_t fo_tab;  // fused output with GroupNorm folding: s, t copied to shared memory (2C floats)
    TokenTable tt;
};

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    // byte offset of 16B chunk `chunk` of a 128-byte row (the TMA 128B swizzle)
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int32_t c0,
                                            int32_t c1, int32_t c2, int32_t c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// 16 bytes global -> shared through the LSU path, zero-filled when !valid
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
// arrives on the mbarrier once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// v0, v1 += x0 * s0 + t0, x1 * s1 + t1 on the packed fp32 pipe (FFMA2 / FADD2)
__device__ __forceinline__ void fma2_acc(float& v0, float& v1, float x0, float x1, float s0, float s1, float t0,
                                         float t1) {
    asm("{\n.reg .b64 X, S, T, V;\n"
        "mov.b64 X, {%2, %3};\nmov.b64 S, {%4, %5};\nmov.b64 T, {%6, %7};\nmov.b64 V, {%0, %1};\n"
        "fma.rn.f32x2 T, X, S, T;\nadd.rn.f32x2 V, V, T;\nmov.b64 {%0, %1}, V;\n}"
        : "+f"(v0), "+f"(v1)
        : "f"(x0), "f"(x1), "f"(s0), "f"(s1), "f"(t0), "f"(t1));
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0), "r"(r1),
                 "r"(r2), "r"(r3)
                 : "memory");
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// hi = RN(x), lo = RN(x - hi), two values at a time
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = pack_bf16(a - __low2float(h), b - __high2float(h));
}

// Shared memory (bytes). RP = K/V tile rows (NTL * 8, a multiple of 16); PL = planes.
//   ring[NS] : FIFO of stages in the consumers' order: per (item, head) nch S-phase stages
//              [Q planes: PL x 32 x 128 B | K planes: PL x RP x 128 B], then ceil(nch / VPS)
//              PV-phase stages of VPS V chunks [PL x RP x 128 B each] (stages 1 KB aligned)
//   sp       : S (fp32), 32 x SP
//   pb       : P (bf16, PL planes), ceil(RP/64) blocks of 32 x 128 B (swizzled rows)
//   ost      : per-warp ctx staging (16 rows)
//   bars     : full[NS], empty[NS]
// One FIFO keeps a fixed prefetch distance across phases and items: V chunks load during the
// softmax, the next item's Q/K chunks during the PV phase. Several CTAs per SM interleave
// their phases, so the memory pipe never drains.
template <int NTL, bool SPLIT, int CW>
struct CoreLay {
    VINF_ATTN_WARP_CONSTANTS(CW)
    static constexpr uint32_t RP = NTL * 8;
    static constexpr uint32_t SP = RP + 4;
    static constexpr uint32_t PL = SPLIT ? 2 : 1;
    static constexpr bool PREG = NTL <= 8;  // P fragments held in registers for PV
    static constexpr uint32_t KT = RP * 128;
    static constexpr uint32_t VPS = (kQT + KT) / KT;  // V chunks per stage
    static constexpr uint32_t ST = (PL * (kQT + KT) + 1023) / 1024 * 1024;
    static constexpr uint32_t PB = ((RP + 63) / 64) * kQBlock * 128;
    static constexpr uint32_t OST = PL * 16 * kOPitch;
    static constexpr uint32_t scratch = (kQBlock * SP * 4 + PL * PB + kConsumerWarps * OST + 127) / 128 * 128;
    // as many CTAs per SM (up to 4) as leave a ring of >= 4 stages each
    static constexpr int pick_ctas() {
        for (int c = 4; c > 1; --c)
            if (c * (scratch + 4 * ST + 2048) <= 226u * 1024u) return c;
        return 1;
    }
    // measured (scripts/attn_micro.py): 3 CTAs per SM for bf16 (deeper rings beat a fourth
    // CTA on long clips, equal at cfg2), 2 for the split mode
    static constexpr int ctas = pick_ctas() < (SPLIT ? 2 : 3) ? pick_ctas() : (SPLIT ? 2 : 3);
    // scratch first, then the ring (NS stages, chosen at launch), then its barriers
    static constexpr uint32_t sp = 0;
    static constexpr uint32_t pb = sp + kQBlock * SP * 4;
    static constexpr uint32_t ost = pb + PL * PB;
    static constexpr uint32_t ring = (ost + kConsumerWarps * OST + 1023) / 1024 * 1024;
    static constexpr uint32_t bars(int ns) { return ring + uint32_t(ns) * ST; }
    static constexpr uint32_t total(int ns) { return bars(ns) + 2u * uint32_t(ns) * 8u + 1024u; }
    // the deepest ring (<= 16 stages) that lets `c` CTAs share an SM (228 KB per SM, of which
    // the driver reserves 1 KB per CTA: sized against 227 KB / c, a ring could leave room for
    // one CTA fewer, as it did for the F = 96, 20 x 32 case: 187 -> 124 us)
    static constexpr int stages(int c, uint32_t extra = 0) {
        int ns = 16;
        while (ns > 2 && uint32_t(c) * (total(ns) + extra + 1024u) > 228u * 1024u) --ns;
        return ns;
    }
    static_assert(total(2) <= 227 * 1024, "attention core shared memory");
};

// Position in a ring of N stages: slot and the parity of its current use.
struct Ring {
    uint32_t n, slot = 0, phase = 0;
    __device__ explicit Ring(uint32_t stages) : n(stages) {}
    __device__ __forceinline__ void next() {
        if (++slot == n) {
            slot = 0;
            phase ^= 1u;
        }
    }
};

// D > 0: the head dim fixed at compile time with heads == 1 (d == C; the chunk loops unroll and
// every chunk is full when D % 64 == 0), D == 0: any configuration
// D > 0 instances also carry a copy warp (warp CW + 1) that loads the Q rows with cp.async
// (a.qfeed): the TMA engine's per-row cost bounds the feed, and the LSU path runs beside it.
template <int NTL, bool SPLIT, int CW, int D>
__global__ void __launch_bounds__((CW + 1 + (D > 0)) * 32, CoreLay<NTL, SPLIT, CW>::ctas)
    attention_core_kernel(const __grid_constant__ AttnMaps maps, const AttnArgs a) {
    using LL = CoreLay<NTL, SPLIT, CW>;
    constexpr int kConsumerWarps = LL::kConsumerWarps, kThreads = LL::kThreads + (D > 0 ? 32 : 0), kWQ = LL::kWQ,
                  kON = LL::kON;
    constexpr uint32_t kOPitch = LL::kOPitch;
    constexpr uint32_t RP = LL::RP;
    constexpr int SP = int(LL::SP);
    const uint32_t NS = a.ns;
    constexpr uint32_t kVPS = LL::VPS;
    constexpr int KC = (int(RP) + 31) / 32;     // softmax columns per lane
    constexpr int NJ = (NTL + kWQ - 1) / kWQ;  // S n8 tiles per warp
    constexpr int NA = NJ <= 2 ? 2 : 1;         // S accumulators per tile (shorter MMA chains)
    static_assert(NTL % 2 == 0 && RP <= uint32_t(kKvMax), "K/V rows padded to a multiple of 16");
    static_assert(D == 0 || RP <= 64, "copy-warp instances: K/V tiles of up to 64 rows");
    extern __shared__ uint8_t sm_raw[];
    // 1 KB aligned, offset from the __shared__ array itself so every access stays a shared-space
    // access (a pointer rebuilt from an integer would make them generic loads / stores)
    uint8_t* sm = sm_raw + ((1024u - (dev::smem_u32(sm_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = dev::smem_u32(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + LL::bars(int(NS)));
    uint64_t* empty = full + NS;
    // the ring's barriers as shared-space addresses (slot s at + 8 s)
    const uint32_t fa = dev::smem_u32(full), ea = fa + 8u * NS;
    float* sp = reinterpret_cast<float*>(sm + LL::sp);

    // zero the ring and scratch once: rows no load of an item writes (K/V padding rows, Q rows
    // past the block) then always hold finite values, and P = 0 meets finite V rows
    for (uint32_t i = tid * 16; i < LL::bars(int(NS)); i += kThreads * 16)
        *reinterpret_cast<uint4*>(sm + i) = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (uint32_t s = 0; s < NS; ++s) {
            dev::mbar_init(&full[s], 1 + (D > 0 && a.qfeed ? 32 : 0));
            dev::mbar_init(&empty[s], kConsumerWarps);
        }
        dev::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeroed smem before TMA writes
    __syncthreads();
    dev::pdl_wait();
    dev::pdl_trigger();
    // fused output: the residual's per-channel scale and shift, after the ring's barriers
    float* stab = reinterpret_cast<float*>(sm + LL::bars(int(NS)) + 2 * NS * 8);
    if (a.fo_tab) {
        for (uint32_t i = tid; i < a.C; i += kThreads) {
            stab[i] = a.fo.s[i];
            stab[a.C + i] = a.fo.t[i];
        }
        __syncthreads();
    }

    constexpr bool kFixed = D > 0;
    const uint32_t heads = kFixed ? 1u : a.heads, nch = kFixed ? uint32_t((D + kDC - 1) / kDC) : a.nch;
    // fused output through the ring (copy-warp instances): each PV stage carries one V chunk
    // (K slot) and the matching residual chunk of the block's queries (Q slot), the residual
    // loaded by the copy warp; the consumers add it from shared memory
    const bool fr = D > 0 && !SPLIT && a.qfeed && a.fo.y != nullptr && a.fo.res_bf16;
    const uint32_t VPS = fr ? 1u : kVPS;
    const uint32_t nvs = (nch + VPS - 1) / VPS;
    const uint32_t dd = kFixed ? uint32_t(D) : a.d, CC = kFixed ? uint32_t(D) : a.C;
    if (D > 0 && warp == kConsumerWarps + 1) {
        // ------ copy warp: the Q rows of every S-phase stage (and the residual chunks) ------
        // lane: 16-byte piece lane & 7 of rows lane >> 3, +4, ...; destination in the TMA
        // 128B-swizzle order the consumers read; one arrival per lane per stage.
        if (!a.qfeed) return;
        Ring r(NS);
        const uint32_t piece = uint32_t(lane) & 7u, r0 = uint32_t(lane) >> 3;
        for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x) {
            const uint32_t p = item / a.nqb, qb = item - p * a.nqb;
            const uint32_t a0 = qb * kQBlock;
            const uint32_t nqh = min(uint32_t(kQBlock), a.nq - a0);
            for (uint32_t h = 0; h < heads; ++h) {
                for (uint32_t ch = 0; ch < nch; ++ch, r.next()) {
                    dev::mbar_wait_a(ea + 8u * r.slot, r.phase ^ 1u);
                    const uint32_t bar = fa + 8u * r.slot;
                    if (a.load_only == 3) {  // diagnostics: the consumers alone
                        dev::mbar_arrive_a(bar);
                        continue;
                    }
                    const uint32_t st = sbase + LL::ring + r.slot * LL::ST;
                    const bool valid = ch * kDC + piece * 8 < dd;
                    for (uint32_t row = r0; row < nqh; row += 4) {
                        // frame-major [frames][HW][3C]: query frame q_frame0 + a0 + row, position p
                        const uint64_t off = (uint64_t(a.q_frame0 + a0 + row) * a.HW + p) * (3ull * CC) + h * dd +
                                             (valid ? ch * kDC + piece * 8 : 0);
                        const uint32_t dst = st + swz(row, piece);
                        cp_async16(dst, a.q + off, valid);
                        if (SPLIT) cp_async16(dst + kQT, a.q_lo + off, valid);
                    }
                    cp_async_arrive(bar);
                }
                for (uint32_t vs = 0; vs < nvs; ++vs, r.next()) {
                    dev::mbar_wait_a(ea + 8u * r.slot, r.phase ^ 1u);
                    const uint32_t bar = fa + 8u * r.slot;
                    if (fr && a.load_only != 3) {  // residual chunk vs (bf16) of the block's query rows -> the Q slot
                        const uint32_t st = sbase + LL::ring + r.slot * LL::ST;
                        const bool valid = vs * kDC + piece * 8 < dd;
                        for (uint32_t row = r0; row < nqh; row += 4)
                            cp_async16(st + swz(row, piece),
                                       static_cast<const __nv_bfloat16*>(a.fo.res) +
                                           (uint64_t(a0 + row) * a.HW + p) * CC + (valid ? vs * kDC + piece * 8 : 0),
                                       valid);
                        cp_async_arrive(bar);
                    } else {
                        dev::mbar_arrive_a(bar);
                    }
                }
            }
        }
        return;
    }
    if (warp == kConsumerWarps) {
        // ---------------- producer: one thread issues every TMA load ----------------
        if (lane != 0) return;
        for (int pl = 0; pl < int(LL::PL); ++pl) dev::tma_prefetch_desc(&maps.g4[pl]);
        Ring r(NS);
        for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x) {
            const uint32_t p = item / a.nqb, qb = item - p * a.nqb;
            const uint32_t nb = a.tt.kv_nbox[qb];
            const uint32_t kvb = uint32_t(a.tt.kv_load_rows[qb]) * 128u * LL::PL;
            const uint32_t* prog = a.tt.kv_box + size_t(qb) * kKvMax;
            const uint32_t nqh = min(uint32_t(kQBlock), a.nq - qb * kQBlock);
            const int32_t qf = int32_t(a.q_frame0 + qb * kQBlock);
            // box: `rows` frames from f0 of 64-wide chunk ch of (which, head h) at position p, over
            // the frame-major [frames][HW][3 x heads][d] buffer; gathers: 2-D row f * HW + p
            auto box4 = [&](uint32_t dst, const CUtensorMap* map, uint32_t bar, uint32_t which, uint32_t h,
                            uint32_t ch, uint32_t f0) {
                tma_load_4d(dst, map, bar, int32_t(ch * kDC), int32_t(which * heads + h), int32_t(p), int32_t(f0));
            };
            // K or V chunk ch (which = 1 / 2) of head h into the stage at dst
            auto load_kv = [&](uint32_t dst, uint32_t bar, uint32_t which, uint32_t h, uint32_t ch) {
                for (uint32_t b = 0; b < nb; ++b) {
                    const uint32_t e = prog[b];
                    const uint32_t row = (e >> 16) & 0xFFu, kind = e >> 24;
                    if (kind == uint32_t(kBoxGather4)) {
                        const uint32_t e1 = prog[b + 1], e2 = prog[b + 2];
                        b += 2;
                        const int32_t col = int32_t(which * CC + h * dd + ch * kDC);
                        auto gr = [&](uint32_t f) { return int32_t(f * a.HW + p); };
                        for (uint32_t pl = 0; pl < LL::PL; ++pl)
                            dev::tma_gather4(dst + pl * LL::KT + row * 128u, &maps.g4[pl], bar, col, gr(e & 0xFFFFu),
                                             gr(e1 & 0xFFFFu), gr(e1 >> 16), gr(e2 & 0xFFFFu));
                        continue;
                    }
                    for (uint32_t pl = 0; pl < LL::PL; ++pl)
                        box4(dst + pl * LL::KT + row * 128u, &maps.box[pl][kind], bar, which, h, ch, e & 0xFFFFu);
                }
            };
            const bool qtma = !(D > 0 && a.qfeed);  // Q rows by TMA here (else the copy warp)
            for (uint32_t h = 0; h < heads; ++h) {
                for (uint32_t ch = 0; ch < nch; ++ch, r.next()) {  // S phase: Q + K chunk
                    dev::mbar_wait_a(ea + 8u * r.slot, r.phase ^ 1u);
                    const uint32_t bar = fa + 8u * r.slot;
                    if (a.load_only == 3) {  // diagnostics: no loads at all (the consumers alone)
                        dev::mbar_arrive_a(bar);
                        continue;
                    }
                    dev::mbar_arrive_expect_tx_a(bar, kvb + (qtma ? nqh * 128u * LL::PL : 0u));
                    const uint32_t st = sbase + LL::ring + r.slot * LL::ST;
                    if (a.fo.y && !fr && h == 0 && ch == 0) {  // fused output: the item's residual rows into L2
                        const uint32_t rb = CC * (a.fo.res_bf16 ? 2u : 4u);
                        const uint8_t* res = static_cast<const uint8_t*>(a.fo.res);
                        for (uint32_t q = 0; q < nqh; ++q)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                             res + (uint64_t(qb * kQBlock + q) * a.HW + p) * rb),
                                         "r"(rb)
                                         : "memory");
                    }
                    // the block's query rows exactly, one box (unless the copy warp loads them)
                    if (qtma)
                        for (uint32_t pl = 0; pl < LL::PL; ++pl)
                            box4(st + pl * kQT, &maps.box[pl][nqh - 1], bar, 0, h, ch, uint32_t(qf));
                    load_kv(st + LL::PL * kQT, bar, 1, h, ch);
                }
                for (uint32_t vs = 0; vs < nvs; ++vs, r.next()) {  // PV phase: VPS V chunks
                    const uint32_t n = min(VPS, nch - vs * VPS);
                    dev::mbar_wait_a(ea + 8u * r.slot, r.phase ^ 1u);
                    const uint32_t bar = fa + 8u * r.slot;
                    if (a.load_only == 3) {
                        dev::mbar_arrive_a(bar);
                        continue;
                    }
                    dev::mbar_arrive_expect_tx_a(bar, kvb * n);
                    const uint32_t st = sbase + LL::ring + r.slot * LL::ST;
                    if (fr) {  // the V chunk into the K slot (the copy warp fills the Q slot)
                        load_kv(st + LL::PL * kQT, bar, 2, h, vs);
                        continue;
                    }
                    for (uint32_t i = 0; i < n; ++i) load_kv(st + i * LL::PL * LL::KT, bar, 2, h, vs * VPS + i);
                }
            }
        }
        return;
    }

    // ---------------- consumers: warps 0 .. kConsumerWarps-1 ----------------
    const int mt = warp & 1, wq = warp >> 1;  // m tile (16 queries), column group
    const uint32_t r7 = lane & 7, hb = lane >> 4, b1 = (lane >> 3) & 1;
    uint32_t a_off[4], b_off[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        a_off[kk] = (mt * 16 + r7 + b1 * 8) * 128 + (((kk * 2 + hb) ^ r7) << 4);
        b_off[kk] = LL::PL * kQT + r7 * 128 + (((kk * 2 + b1) ^ r7) << 4);
    }
    // V fragments (ldmatrix.trans) of n8 tiles kON*wq + 2i + {0, 1}, within a V chunk
    uint32_t v_off[kON / 2];
#pragma unroll
    for (int i = 0; i < kON / 2; ++i)
        v_off[i] = (r7 + b1 * 8) * 128 + (((uint32_t(kON * wq + 2 * i) + hb) ^ r7) << 4);
    const int g = lane >> 2, t4 = lane & 3;
    auto p_addr = [&](int kq) {  // P fragment (A operand) of k16 step kq, plane 0
        return sbase + LL::pb + uint32_t(kq >> 2) * (kQBlock * 128) + (mt * 16 + r7 + b1 * 8) * 128 +
               ((((kq & 3) * 2 + hb) ^ r7) << 4);
    };
    const float bw = a.tt.wflag ? a.bias : 0.f, bg = a.tt.gflag ? a.bias : 0.f;
    const uint64_t ldc = CC;
    uint8_t* ost = sm + LL::ost + warp * LL::OST;
    Ring r(NS);
    if (a.load_only == 1) {  // diagnostics: the producer's feed rate alone
        for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x)
            for (uint32_t k = 0; k < heads * (nch + nvs); ++k, r.next()) {
                dev::mbar_wait_a(fa + 8u * r.slot, r.phase);
                __syncwarp();
                if (lane == 0) dev::mbar_arrive_a(ea + 8u * r.slot);
            }
        return;
    }
    for (uint32_t item = blockIdx.x; item < a.items; item += gridDim.x) {
        const uint32_t p = item / a.nqb, qb = item - p * a.nqb;
        const uint32_t a0 = qb * kQBlock;
        const uint32_t nqh = min(uint32_t(kQBlock), a.nq - a0);
        const uint32_t R = a.tt.kv_count[qb];
        const uint8_t* gm = a.tt.gmult + size_t(qb) * kKvMax;
        int ngc[KC];  // global tokens on this lane's columns (the same for every query of the block)
#pragma unroll
        for (int k = 0; k < KC; ++k) ngc[k] = lane + 32 * k < int(R) ? gm[lane + 32 * k] : 0;
        // window column ranges of this warp's softmax rows warp + kConsumerWarps * i, read
        // once per item (their latency hides under the S phase)
        // narrow tiles (quad softmax): this thread's row tid / 4 and its eight columns
        int qlo = 0, qhi = -1, qng[8];
        if constexpr (RP <= 32 && kConsumerWarps == 4) {
            const uint32_t rr = uint32_t(tid) >> 2, quarter = uint32_t(lane) & 3u;
            if (rr < nqh) {
                qlo = a.tt.wlo[a0 + rr];
                qhi = a.tt.whi[a0 + rr];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t c = quarter * 8 + uint32_t(k);
                qng[k] = c < R ? gm[c] : 0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) qng[k] = 0;
        }
        constexpr int kRows = kQBlock / kConsumerWarps;
        uint32_t wl[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const uint32_t rr = warp + kConsumerWarps * i;
            wl[i] = rr < nqh ? uint32_t(a.tt.wlo[a0 + rr]) | uint32_t(a.tt.whi[a0 + rr]) << 8 : 0u;
        }
        for (uint32_t h = 0; h < heads; ++h) {
            // ---------------- S = Q K^T ----------------
            // warp: m tile mt (16 queries) x n8 tiles wq, wq + kWQ, ... of the RP key columns
            float acc[NJ][NA][4];
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int x = 0; x < NA; ++x) acc[j][x][0] = acc[j][x][1] = acc[j][x][2] = acc[j][x][3] = 0.f;
            for (uint32_t ch = 0; ch < nch; ++ch, r.next()) {
                dev::mbar_wait_a(fa + 8u * r.slot, r.phase);
                const uint32_t st = sbase + LL::ring + r.slot * LL::ST;
                const uint32_t vw = min(uint32_t(kDC), dd - ch * kDC);
#pragma unroll
                for (int kk = 0; kk < kDC / 16; ++kk) {
                    if (kk * 16 >= int(vw)) break;  // zero-filled past the head dim
                    uint32_t qa[4], ql[4];
                    ldsm_x4(st + a_off[kk], qa);
                    if (SPLIT) ldsm_x4(st + kQT + a_off[kk], ql);
                    if constexpr (!SPLIT && NJ % 2 == 0 && NTL == NJ * kWQ) {
                        // two n8 key tiles per ldmatrix.x4 (lanes 16-31 address the second)
#pragma unroll
                        for (int j = 0; j < NJ; j += 2) {
                            uint32_t kf[4];
                            ldsm_x4(st + b_off[kk] + (wq + kWQ * (j + int(hb))) * 1024, kf);
                            mma_bf16(acc[j][NA == 2 ? (kk & 1) : 0], qa, kf[0], kf[1]);
                            mma_bf16(acc[j + 1][NA == 2 ? (kk & 1) : 0], qa, kf[2], kf[3]);
                        }
                        continue;
                    }
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        if (wq + kWQ * j < NTL) {
                            float(&c)[4] = acc[j][NA == 2 ? (kk & 1) : 0];
                            uint32_t k0, k1;
                            ldsm_x2(st + b_off[kk] + (wq + kWQ * j) * 1024, k0, k1);
                            mma_bf16(c, qa, k0, k1);
                            if (SPLIT) {
                                uint32_t l0, l1;
                                ldsm_x2(st + LL::KT + b_off[kk] + (wq + kWQ * j) * 1024, l0, l1);
                                mma_bf16(c, qa, l0, l1);
                                mma_bf16(c, ql, k0, k1);
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) dev::mbar_arrive_a(ea + 8u * r.slot);
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int nt = wq + kWQ * j;
                if (nt < NTL) {
                    float v[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = NA == 2 ? acc[j][0][e] + acc[j][NA - 1][e] : acc[j][0][e];
                    const int col = nt * 8 + t4 * 2;
                    *reinterpret_cast<float2*>(&sp[(mt * 16 + g) * SP + col]) = make_float2(v[0], v[1]);
                    *reinterpret_cast<float2*>(&sp[(mt * 16 + g + 8) * SP + col]) = make_float2(v[2], v[3]);
                }
            }
            dev::named_bar(1, kConsumerWarps * 32);
            // ---------------- softmax over the token lists, per row -> P (bf16) ----------
            // Column c of the block's K/V list carries query qa's window token iff
            // wlo <= c <= whi, and gmult[c] global tokens; p_c = [window] e^(l_w - m) +
            // gmult[c] e^(l_g - m), summed one token at a time. A warp owns whole rows.
            if constexpr (RP <= 32 && kConsumerWarps == 4) {
                // narrow tiles: all 32 rows in one pass, four threads per row (eight columns
                // each, two quad shuffles per reduction), P written as one 16-byte piece per thread
                const uint32_t rr = uint32_t(tid) >> 2, quarter = uint32_t(lane) & 3u;
                if (rr < nqh) {
                    const float* row = sp + rr * SP + quarter * 8;
                    const bool have = quarter * 8 < RP;  // columns past RP were never stored
                    const float4 s0 = have ? *reinterpret_cast<const float4*>(row) : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 s1 = have ? *reinterpret_cast<const float4*>(row + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float sr[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
                    float sv[8], m = -INFINITY;
                    bool inw[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int c = int(quarter) * 8 + k;
                        const bool ok = c < int(R);
                        sv[k] = ok ? a.scale * sr[k] : 0.f;
                        inw[k] = ok && c >= qlo && c <= qhi;
                        if (inw[k]) m = fmaxf(m, sv[k] + bw);
                        if (qng[k]) m = fmaxf(m, sv[k] + bg);
                    }
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
                    float e[8], z = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        e[k] = inw[k] ? (SPLIT ? expf(sv[k] + bw - m) : __expf(sv[k] + bw - m)) : 0.f;
                        if (qng[k]) e[k] += float(qng[k]) * (SPLIT ? expf(sv[k] + bg - m) : __expf(sv[k] + bg - m));
                        z += e[k];
                    }
                    z += __shfl_xor_sync(0xffffffffu, z, 1);
                    z += __shfl_xor_sync(0xffffffffu, z, 2);
                    const float zi = 1.0f / z;
                    uint32_t ph[4], pl[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (SPLIT)
                            split2(e[2 * k] * zi, e[2 * k + 1] * zi, ph[k], pl[k]);
                        else
                            ph[k] = pack_bf16(e[2 * k] * zi, e[2 * k + 1] * zi);
                    }
                    *reinterpret_cast<uint4*>(sm + LL::pb + swz(rr, quarter)) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
                    if (SPLIT)
                        *reinterpret_cast<uint4*>(sm + LL::pb + LL::PB + swz(rr, quarter)) =
                            make_uint4(pl[0], pl[1], pl[2], pl[3]);
                } else {
                    // keep the quad's shuffles converged (rows past the block contribute nothing)
                    float m = 0.f;
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
                    m += __shfl_xor_sync(0xffffffffu, m, 1);
                    m += __shfl_xor_sync(0xffffffffu, m, 2);
                }
            } else
            // two rows per pass (independent shuffle chains); the block's global-token
            // multiplicities per column were read once per item (ngc)
#pragma unroll
            for (int i0 = 0; i0 < kRows; i0 += 2) {
                const uint32_t r0 = warp + kConsumerWarps * i0, r1 = r0 + kConsumerWarps;
                if (r0 >= nqh) break;
                const bool two = r1 < nqh;
                float sv[2][KC], pv[2][KC], m[2] = {-INFINITY, -INFINITY}, z[2] = {0.f, 0.f};
                bool inw[2][KC];
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    const uint32_t rr = w ? (two ? r1 : r0) : r0;
                    const float* row = sp + rr * SP;
                    const uint32_t wlh = (w && two) ? wl[(i0 + 1) % kRows] : wl[i0];
                    const int lo = int(wlh & 0xFFu), hi = int(wlh >> 8);
#pragma unroll
                    for (int k = 0; k < KC; ++k) {
                        const int c = lane + 32 * k;
                        const bool ok = c < int(R);
                        sv[w][k] = ok ? a.scale * row[c] : 0.f;
                        inw[w][k] = ok && c >= lo && c <= hi;
                        if (inw[w][k]) m[w] = fmaxf(m[w], sv[w][k] + bw);
                        if (ngc[k]) m[w] = fmaxf(m[w], sv[w][k] + bg);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    m[0] = fmaxf(m[0], __shfl_xor_sync(0xffffffffu, m[0], o));
                    m[1] = fmaxf(m[1], __shfl_xor_sync(0xffffffffu, m[1], o));
                }
#pragma unroll
                for (int w = 0; w < 2; ++w)
#pragma unroll
                    for (int k = 0; k < KC; ++k) {
                        float e = inw[w][k] ? (SPLIT ? expf(sv[w][k] + bw - m[w]) : __expf(sv[w][k] + bw - m[w])) : 0.f;
                        if (ngc[k])  // the column's ngc global tokens, each e^(l_g - m)
                            e += float(ngc[k]) * (SPLIT ? expf(sv[w][k] + bg - m[w]) : __expf(sv[w][k] + bg - m[w]));
                        pv[w][k] = e;
                        z[w] += e;
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    z[0] += __shfl_xor_sync(0xffffffffu, z[0], o);
                    z[1] += __shfl_xor_sync(0xffffffffu, z[1], o);
                }
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    if (w == 1 && !two) break;
                    const uint32_t rr = w ? r1 : r0;
                    const float zi = 1.0f / z[w];
#pragma unroll
                    for (int k = 0; k < KC; ++k) {
                        const uint32_t c = lane + 32 * k;
                        if (c < RP) {
                            const uint32_t off =
                                LL::pb + (c >> 6) * (kQBlock * 128) + swz(rr, (c & 63) >> 3) + (c & 7) * 2;
                            const float v = pv[w][k] * zi;
                            const __nv_bfloat16 vh = __float2bfloat16_rn(v);
                            *reinterpret_cast<__nv_bfloat16*>(sm + off) = vh;
                            if (SPLIT)
                                *reinterpret_cast<__nv_bfloat16*>(sm + off + LL::PB) =
                                    __float2bfloat16_rn(v - __bfloat162float(vh));
                        }
                    }
                }
            }
            dev::named_bar(1, kConsumerWarps * 32);
            // ---------------- ctx = P V ----------------
            // warp: m tile mt, n8 tiles kON*wq .. kON*wq + kON-1 of each 64-wide output chunk;
            // the tile goes through a per-warp staging block to 16-byte row stores
            uint32_t pa[LL::PREG ? NTL / 2 : 1][4], pal[LL::PREG && SPLIT ? NTL / 2 : 1][4];
            if (LL::PREG) {
#pragma unroll
                for (int kq = 0; kq < NTL / 2; ++kq) {
                    ldsm_x4(p_addr(kq), pa[LL::PREG ? kq : 0]);
                    if (SPLIT) ldsm_x4(p_addr(kq) + LL::PB, pal[LL::PREG && SPLIT ? kq : 0]);
                }
            }
            constexpr int kPc = (16 * kON + 31) / 32;  // output pieces per lane per chunk
            for (uint32_t vs = 0; vs < nvs; ++vs, r.next()) {
                dev::mbar_wait_a(fa + 8u * r.slot, r.phase);
                const uint32_t n = min(VPS, nch - vs * VPS);
                // fused output, bf16 residual: this stage's residual pieces requested up front, so
                // their latency (L2: the producer prefetched the item's rows) hides under the PV math
                uint4 rpre[SPLIT ? 1 : kVPS][kPc];
                if (D == 0 && !SPLIT && a.fo.y && a.fo.res_bf16) {
#pragma unroll
                    for (int i = 0; i < int(kVPS); ++i)
#pragma unroll
                        for (int i2 = 0; i2 < kPc; ++i2) {
                            const uint32_t pc = lane + 32 * i2, ch = vs * VPS + uint32_t(i);
                            const uint32_t q = mt * 16 + pc / kON, col = uint32_t(wq) * kON * 8 + (pc % kON) * 8;
                            if (uint32_t(i) < n && pc < uint32_t(16 * kON) && q < nqh && ch * kDC + col < dd)
                                rpre[SPLIT ? 0 : i][i2] = __ldg(reinterpret_cast<const uint4*>(
                                    static_cast<const __nv_bfloat16*>(a.fo.res) +
                                    (uint64_t(a0 + q) * a.HW + p) * ldc + ch * kDC + col));
                        }
                }
#pragma unroll
                for (uint32_t i = 0; i < kVPS; ++i) {
                    if (i >= n) break;
                    const uint32_t ch = vs * VPS + i;
                    const uint32_t slot = LL::ring + r.slot * LL::ST;  // fr: the residual chunk at its start
                    const uint32_t st = sbase + slot + (fr ? LL::PL * kQT : i * LL::PL * LL::KT);
                    const uint32_t vw = min(uint32_t(kDC), dd - ch * kDC);
                    const uint32_t c0w = uint32_t(wq) * kON * 8;  // this warp's first column in the chunk
                    const bool live = c0w < vw;
                    float o[kON][4];
#pragma unroll
                    for (int nn = 0; nn < kON; ++nn) o[nn][0] = o[nn][1] = o[nn][2] = o[nn][3] = 0.f;
                    if (live) {
#pragma unroll
                        for (int kq = 0; kq < NTL / 2; ++kq) {
                            uint32_t pf[4], pfl[4];
                            if (LL::PREG) {
#pragma unroll
                                for (int k = 0; k < 4; ++k) pf[k] = pa[LL::PREG ? kq : 0][k];
                                if (SPLIT)
#pragma unroll
                                    for (int k = 0; k < 4; ++k) pfl[k] = pal[LL::PREG && SPLIT ? kq : 0][k];
                            } else {
                                ldsm_x4(p_addr(kq), pf);
                                if (SPLIT) ldsm_x4(p_addr(kq) + LL::PB, pfl);
                            }
#pragma unroll
                            for (int i2 = 0; i2 < kON / 2; ++i2) {
                                uint32_t b[4];
                                ldsm_x4_t(st + v_off[i2] + kq * 2048, b);
                                mma_bf16(o[2 * i2], pf, b[0], b[1]);
                                mma_bf16(o[2 * i2 + 1], pf, b[2], b[3]);
                                if (SPLIT) {
                                    uint32_t bl[4];
                                    ldsm_x4_t(st + LL::KT + v_off[i2] + kq * 2048, bl);
                                    mma_bf16(o[2 * i2], pf, bl[0], bl[1]);
                                    mma_bf16(o[2 * i2 + 1], pf, bl[2], bl[3]);
                                    mma_bf16(o[2 * i2], pfl, b[0], b[1]);
                                    mma_bf16(o[2 * i2 + 1], pfl, b[2], b[3]);
                                }
                            }
                        }
                        // accumulators -> staging [16 rows][kON*8 cols] (bf16; lo plane after it);
                        // bf16 mode: two n8 tiles per stmatrix.x4
                        if constexpr (!SPLIT && kON % 2 == 0) {
                            const uint32_t mrow = ((uint32_t(lane) >> 3) & 1u) * 8u + (uint32_t(lane) & 7u);
#pragma unroll
                            for (int nn = 0; nn < kON; nn += 2) {
                                const uint32_t addr = dev::smem_u32(ost) + mrow * kOPitch +
                                                      uint32_t(nn + int(uint32_t(lane) >> 4)) * 16u;
                                stsm_x4(addr, pack_bf16(o[nn][0], o[nn][1]), pack_bf16(o[nn][2], o[nn][3]),
                                        pack_bf16(o[nn + 1][0], o[nn + 1][1]), pack_bf16(o[nn + 1][2], o[nn + 1][3]));
                            }
                        } else
#pragma unroll
                        for (int nn = 0; nn < kON; ++nn) {
                            const uint32_t o0 = uint32_t(g) * kOPitch + (nn * 8 + t4 * 2) * 2, o1 = o0 + 8 * kOPitch;
                            if (SPLIT) {
                                uint32_t h0, l0, h1, l1;
                                split2(o[nn][0], o[nn][1], h0, l0);
                                split2(o[nn][2], o[nn][3], h1, l1);
                                *reinterpret_cast<uint32_t*>(ost + o0) = h0;
                                *reinterpret_cast<uint32_t*>(ost + o1) = h1;
                                *reinterpret_cast<uint32_t*>(ost + 16 * kOPitch + o0) = l0;
                                *reinterpret_cast<uint32_t*>(ost + 16 * kOPitch + o1) = l1;
                            } else {
                                *reinterpret_cast<uint32_t*>(ost + o0) = pack_bf16(o[nn][0], o[nn][1]);
                                *reinterpret_cast<uint32_t*>(ost + o1) = pack_bf16(o[nn][2], o[nn][3]);
                            }
                        }
                        __syncwarp();
                        // 16 rows x kON 16-byte pieces: row rr -> query a0 + 16 mt + rr
                        constexpr int kPieces = 16 * kON;
                        // fused output through the ring: this lane's columns are the same for all
                        // of its pieces (kON divides 32), so s and t are read once per chunk
                        float ssc[8], tsc[8];
                        if (fr && a.fo_tab) {
                            const float* sc = stab + ch * kDC + c0w + (uint32_t(lane) % kON) * 8;
                            const float4 s0 = *reinterpret_cast<const float4*>(sc);
                            const float4 s1 = *reinterpret_cast<const float4*>(sc + 4);
                            const float4 t0 = *reinterpret_cast<const float4*>(sc + CC);
                            const float4 t1 = *reinterpret_cast<const float4*>(sc + CC + 4);
                            ssc[0] = s0.x; ssc[1] = s0.y; ssc[2] = s0.z; ssc[3] = s0.w;
                            ssc[4] = s1.x; ssc[5] = s1.y; ssc[6] = s1.z; ssc[7] = s1.w;
                            tsc[0] = t0.x; tsc[1] = t0.y; tsc[2] = t0.z; tsc[3] = t0.w;
                            tsc[4] = t1.x; tsc[5] = t1.y; tsc[6] = t1.z; tsc[7] = t1.w;
                        }
#pragma unroll
                        for (int i2 = 0; i2 < (kPieces + 31) / 32; ++i2) {
                            const uint32_t pc = lane + 32 * i2;
                            const uint32_t rr = pc / kON, part = pc % kON;
                            const uint32_t q = mt * 16 + rr, col = c0w + part * 8;
                            if (pc < uint32_t(kPieces) && q < nqh && col < vw) {
                                const uint64_t o = (uint64_t(a0 + q) * a.HW + p) * ldc + h * dd + ch * kDC + col;
                                const uint4 hv = *reinterpret_cast<const uint4*>(ost + rr * kOPitch + part * 16);
                                if (a.fo.y) {  // y = ctx' + residual (one head: ldc = d)
                                    float v[8];
                                    unpack8(hv, v);
                                    if (SPLIT) {
                                        unpack8_add(*reinterpret_cast<const uint4*>(ost + 16 * kOPitch + rr * kOPitch +
                                                                                     part * 16),
                                                    v);
                                        fuse_o_store(a.fo, o, ch * kDC + col, v);
                                    } else if (fr) {  // the residual piece from the stage's Q slot
                                        const uint4 u = *reinterpret_cast<const uint4*>(sm + slot + swz(q, col >> 3));
                                        if (a.fo_tab) {
                                            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                                            for (int k = 0; k < 4; ++k) {
                                                const float2 x = __bfloat1622float2(u2[k]);
                                                fma2_acc(v[2 * k], v[2 * k + 1], x.x, x.y, ssc[2 * k], ssc[2 * k + 1],
                                                         tsc[2 * k], tsc[2 * k + 1]);
                                            }
                                        } else {
                                            fuse_o_add_bf16(a.fo, u, ch * kDC + col, v);
                                        }
                                        fuse_o_write(a.fo, o, v);
                                    } else if (D == 0 && a.fo.res_bf16) {
                                        fuse_o_add_bf16(a.fo, rpre[SPLIT ? 0 : i][i2], ch * kDC + col, v);
                                        fuse_o_write(a.fo, o, v);
                                    } else {
                                        fuse_o_store(a.fo, o, ch * kDC + col, v);
                                    }
                                } else {
                                    *reinterpret_cast<uint4*>(a.ctx + o) = hv;
                                    if (SPLIT)
                                        *reinterpret_cast<uint4*>(a.ctx + o + a.ctx_lo) = *reinterpret_cast<const uint4*>(
                                            ost + 16 * kOPitch + rr * kOPitch + part * 16);
                                }
                            }
                        }
                        __syncwarp();  // staging is rewritten by the next chunk
                    }
                }
                __syncwarp();
                if (lane == 0) dev::mbar_arrive_a(ea + 8u * r.slot);
            }
        }
    }
}

int g_sms = 0;

// 4-D view of the [frames][HW][3 x heads][d] Q/K/V buffer (one bf16 plane): boxes of
// {64 head-dim elements, 1 head, 1 position, kind + 1 frames}, 128-byte swizzle; head-dim
// elements past d read as zero.
int make_maps(AttnMaps& m, const void* qkv, const void* qkv_lo, uint32_t frames, uint32_t HW, uint32_t C,
              uint32_t heads) {
    auto fn = get_encode_fn();
    if (!fn) return int(cudaErrorNotSupported);
    const uint32_t d = C / heads;
    for (int pl = 0; pl < 2; ++pl) {
        const void* base = pl == 0 ? qkv : qkv_lo;
        for (int k = 0; k < kBoxKinds; ++k) {
            if (!base) {
                m.box[pl][k] = m.box[0][k];
                continue;
            }
            // frame-major [frames][HW][3C] rows (position stride 3C, frame stride HW 3C)
            const uint64_t row = uint64_t(C) * 3 * 2;
            cuuint64_t gdim[4] = {d, 3ull * heads, HW, frames};
            cuuint64_t gstride[3] = {uint64_t(d) * 2, row, row * HW};
            cuuint32_t box[4] = {uint32_t(kDC), 1, 1, uint32_t(k) + 1};
            cuuint32_t estride[4] = {1, 1, 1, 1};
            const CUresult r = fn(&m.box[pl][k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), gdim,
                                  gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
        }
        if (!base) {
            m.g4[pl] = m.g4[0];
            continue;
        }
        cuuint64_t gdim[2] = {3ull * C, uint64_t(HW) * frames};
        cuuint64_t gstride[1] = {uint64_t(C) * 3 * 2};
        cuuint32_t box[2] = {uint32_t(kDC), 1};
        cuuint32_t estride[2] = {1, 1};
        const CUresult r = fn(&m.g4[pl], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                              box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return int(cudaErrorInvalidValue);
    }
    return 0;
}

template <int NTL, bool SPLIT, int CW, int D>
int launch_core(const AttnMaps& maps, AttnArgs args, cudaStream_t s) {
    using LL = CoreLay<NTL, SPLIT, CW>;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(attention_core_kernel<NTL, SPLIT, CW, D>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return int(e);
        attr = true;
    }
    if (g_sms == 0) {
        int dv = 0;
        cudaGetDevice(&dv);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dv);
        if (g_sms <= 0) g_sms = 148;
    }
    // CTAs per SM (VINF_ATTN_CTAS, diagnostics) and the ring depth that fits them
    static const int env_ctas = [] {
        const char* e = getenv("VINF_ATTN_CTAS");
        return e ? atoi(e) : 0;
    }();
    const int ctas = env_ctas >= 1 && env_ctas <= 4 ? env_ctas : LL::ctas;
    // fused output with GroupNorm folding (copy-warp instances): s, t in shared memory
    args.fo_tab = D > 0 && args.fo.y && args.fo.s ? 1u : 0u;
    const uint32_t tab = args.fo_tab ? (2 * args.C * 4 + 127) / 128 * 128 : 0u;
    args.ns = uint32_t(LL::stages(ctas, tab));
    const uint32_t slots = uint32_t(g_sms) * uint32_t(ctas);
    const uint32_t grid = args.items < slots ? args.items : slots;
    static const uint32_t qfeed = [] {
        const char* e = getenv("VINF_ATTN_QFEED");
        return e ? uint32_t(atoi(e) != 0) : 1u;  // 0 = all by TMA, 1 = Q rows by the copy warp
    }();
    args.qfeed = D > 0 ? qfeed : 0u;
    return int(launch_pdl(attention_core_kernel<NTL, SPLIT, CW, D>, dim3(grid), dim3(LL::kThreads + (D > 0 ? 32 : 0)),
                          LL::total(int(args.ns)) + tab, s, maps, args));
}

// four consumer warps per CTA (eight, at 2 CTAs per SM, measured slower on the cfg2 and
// 288-frame shapes and with the fused output: profiles/r02_attn/warps_ctas.txt; removed)
template <int NTL, bool SPLIT>
int launch_ntl(const AttnMaps& maps, const AttnArgs& args, cudaStream_t s) {
    // one head with the head dim of a VideoCrafter2 level: compile-time chunk loops and the
    // copy warp (a fused output goes through the ring only with the copy warp: without it,
    // VINF_ATTN_QFEED=0, the generic instance, whose consumers load the residual themselves)
    static const bool qfeed = [] {
        const char* q = getenv("VINF_ATTN_QFEED");
        return !q || atoi(q) != 0;
    }();
    if constexpr (NTL <= 8 && !SPLIT) {
        if (args.heads == 1 && (!args.fo.y || (qfeed && args.fo.res_bf16))) switch (args.d) {
                case 320: return launch_core<NTL, SPLIT, 4, 320>(maps, args, s);
                case 640: return launch_core<NTL, SPLIT, 4, 640>(maps, args, s);
                case 1280: return launch_core<NTL, SPLIT, 4, 1280>(maps, args, s);
                default: break;
            }
    }
    return launch_core<NTL, SPLIT, 4, 0>(maps, args, s);
}

template <bool SPLIT>
int launch_mode(uint32_t RP, const AttnMaps& maps, const AttnArgs& args, cudaStream_t s) {
#define CORE(NTL) \
    case NTL * 8: \
        return launch_ntl<NTL, SPLIT>(maps, args, s)
    switch (RP) {
        CORE(2); CORE(4); CORE(6); CORE(8); CORE(10); CORE(12);
        CORE(14); CORE(16); CORE(18); CORE(20); CORE(22); CORE(24);
        default: return int(cudaErrorInvalidValue);
    }
#undef CORE
}

}  // namespace

bool attention_core_supported(uint32_t C, uint32_t heads, const TokenTable& tt) {
    return heads > 0 && C % heads == 0 && (C / heads) % 8 == 0 && tt.kv_ok && tt.max_kv > 0 &&
           tt.max_kv <= kKvMax;
}

int launch_attention_core(const void* qkv, const void* qkv_lo, uint32_t qkv_frames, uint32_t HW, uint32_t C,
                          uint32_t heads, uint32_t nq, uint32_t q_frame0, const TokenTable& tt, float scale,
                          float bias, void* ctx, void* ctx_lo, cudaStream_t s, const FuseO* fo) {
    if (HW == 0 || !qkv || !ctx || (qkv_lo == nullptr) != (ctx_lo == nullptr)) return int(cudaErrorInvalidValue);
    if (fo && fo->y && (heads != 1 || !fo->res || (fo->s == nullptr) != (fo->t == nullptr)))
        return int(cudaErrorInvalidValue);
    if (nq == 0) return 0;
    if (!attention_core_supported(C, heads, tt)) return int(cudaErrorInvalidValue);
    if (reinterpret_cast<uintptr_t>(qkv) % 16 || reinterpret_cast<uintptr_t>(qkv_lo) % 16)
        return int(cudaErrorInvalidValue);
    // Which ring feeds the core (same arithmetic and token rules; measured on one B200,
    // profiles/r02_attn/impl_ab.txt): the TMA ring for bf16 blocks of <= 32 distinct K/V frames
    // (the 24-frame VideoCrafter2 clip: 72.7 vs 77.1 us), the cp.async ring of one position per
    // CTA everywhere else (wide tiles of long clips: 581 vs 784 us at F = 288, C = 320; the
    // split mode: 144 vs 154 us), where thread-issued copies of many CTAs keep more in flight.
    const uint32_t RPw = (uint32_t(tt.max_kv) + 15) & ~15u;
    // Single-head VideoCrafter2 head dims on a one-block clip (nq <= 32: a clip-parallel worker's
    // 24 frames) run the copy-warp TMA instances up to 64 K/V rows (its halo + remote-global
    // list: 124 vs 148 us for 2 workers, 139 vs 152 us for 8, profiles/r02_attn/worker_impl.txt);
    // long clips (many blocks per position) keep the cp.async ring above 32 rows (626 vs 862 us
    // at F = 288, C = 320).
    const bool cw_inst = heads == 1 && (C == 320 || C == 640 || C == 1280) && nq <= uint32_t(kQBlock);
    const int impl = g_attn_impl ? g_attn_impl : (!qkv_lo && (RPw <= 32 || (cw_inst && RPw <= g_cw_rows)) ? 1 : 2);
    if (impl == 2)
        return launch_attention_core_cpasync(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s,
                                             fo);
    // 66 tensor maps per buffer: encoded once per (buffer, shape), then reused
    struct Cached {
        const void *q = nullptr, *ql = nullptr;
        uint32_t frames = 0, HW = 0, C = 0, heads = 0;
        int layout = -1;
        AttnMaps maps;
    };
    static std::mutex mu;
    static Cached cache[8];
    static int cache_next = 0;
    AttnMaps maps;
    {
        std::lock_guard<std::mutex> g(mu);
        int hit = -1;
        for (int i = 0; i < 8; ++i) {
            const Cached& c = cache[i];
            if (c.q == qkv && c.ql == qkv_lo && c.frames == qkv_frames && c.HW == HW && c.C == C && c.heads == heads &&
                true)
                hit = i;
        }
        if (hit < 0) {
            Cached& c = cache[cache_next];
            c.layout = -1;
            const int rc = make_maps(c.maps, qkv, qkv_lo, qkv_frames, HW, C, heads);
            if (rc) return rc;
            c.q = qkv;
            c.ql = qkv_lo;
            c.frames = qkv_frames;
            c.HW = HW;
            c.C = C;
            c.heads = heads;
            c.layout = 0;
            hit = cache_next;
            cache_next = (cache_next + 1) % 8;
        }
        maps = cache[hit].maps;
    }
    AttnArgs args;
    args.HW = HW;
    args.C = C;
    args.heads = heads;
    args.d = C / heads;
    args.nch = (args.d + kDC - 1) / kDC;
    args.nq = nq;
    args.nqb = (nq + kQBlock - 1) / kQBlock;
    args.q_frame0 = q_frame0;
    args.items = HW * args.nqb;
    static const uint32_t load_only = getenv("VINF_ATTN_LOAD_ONLY") ? uint32_t(atoi(getenv("VINF_ATTN_LOAD_ONLY"))) : 0u;
    args.load_only = load_only;
    args.q = static_cast<const __nv_bfloat16*>(qkv);
    args.q_lo = static_cast<const __nv_bfloat16*>(qkv_lo);
    args.scale = scale;
    args.bias = bias;
    args.ctx = static_cast<__nv_bfloat16*>(ctx);
    args.ctx_lo = ctx_lo ? static_cast<__nv_bfloat16*>(ctx_lo) - static_cast<__nv_bfloat16*>(ctx) : 0;
    args.tt = tt;
    if (fo) args.fo = *fo;
    const uint32_t RP = (uint32_t(tt.max_kv) + 15) & ~15u;
    return qkv_lo ? launch_mode<true>(RP, maps, args, s) : launch_mode<false>(RP, maps, args, s);
}

namespace {
__global__ void read_bw_kernel(const uint4* __restrict__ p, uint64_t n, uint32_t* sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}
// 1-D bulk copies of `chunk` bytes into a ring of `stages` smem slots, one issuing thread
// per CTA, the CTA's 4 other warps release the slots (the shape of the attention core's feed).
__global__ void __launch_bounds__(160) bulk_bw_kernel(const uint8_t* __restrict__ p, uint64_t bytes, uint32_t chunk,
                                                        uint32_t stages) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * chunk);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            dev::mbar_init(&full[s], 1);
            dev::mbar_init(&empty[s], 4);
        }
        dev::fence_barrier_init();
    }
    __syncthreads();
    const uint64_t n = bytes / chunk;
    Ring r(stages);
    if (warp == 4) {
        if (lane) return;
        for (uint64_t i = blockIdx.x; i < n; i += gridDim.x, r.next()) {
            dev::mbar_wait(&empty[r.slot], r.phase ^ 1u);
            dev::mbar_arrive_expect_tx(&full[r.slot], chunk);
            dev::bulk_g2s(dev::smem_u32(sm + r.slot * chunk), p + i * chunk, chunk, &full[r.slot]);
        }
        return;
    }
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x, r.next()) {
        dev::mbar_wait(&full[r.slot], r.phase);
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&empty[r.slot]);
    }
}
}  // namespace

// Diagnostics: the feed above over `bytes` with ctas CTAs per SM (average ms).
int bulk_bw_bench(uint64_t bytes, uint32_t chunk, uint32_t stages, uint32_t ctas, int iters, float* ms) {
    void* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return int(cudaErrorMemoryAllocation);
    cudaMemset(buf, 1, bytes);
    if (g_sms == 0) cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t smem = stages * chunk + stages * 16 + 64;
    cudaFuncSetAttribute(bulk_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bulk_bw_kernel<<<g_sms * ctas, 160, smem>>>(static_cast<const uint8_t*>(buf), bytes, chunk, stages);
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i)
        bulk_bw_kernel<<<g_sms * ctas, 160, smem>>>(static_cast<const uint8_t*>(buf), bytes, chunk, stages);
    cudaEventRecord(b);
    const cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    *ms = t / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    return int(e);
}

// Diagnostics: streaming 16-byte loads over `bytes` (average ms over iters).
int read_bw_bench(uint64_t bytes, int iters, float* ms) {
    void* buf = nullptr;
    if (cudaMalloc(&buf, bytes + 64) != cudaSuccess) return int(cudaErrorMemoryAllocation);
    cudaMemset(buf, 1, bytes + 64);
    if (g_sms == 0) cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t n = bytes / 16;
    read_bw_kernel<<<g_sms * 8, 256>>>(static_cast<const uint4*>(buf), n, static_cast<uint32_t*>(buf) + bytes / 4);
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i)
        read_bw_kernel<<<g_sms * 8, 256>>>(static_cast<const uint4*>(buf), n, static_cast<uint32_t*>(buf) + bytes / 4);
    cudaEventRecord(b);
    const cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    *ms = t / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    return int(e);
}

}  // namespace vinf
