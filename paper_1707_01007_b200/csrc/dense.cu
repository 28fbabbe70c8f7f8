// Dense (tensor-core) closure iteration for sm_100a: tcgen05 int8 MMA on 0/1 tiles.
//
// One Jacobi loop body of Algorithm 1, T_k = T_{k-1} ∪ (T_{k-1} × T_{k-1}), with
// the product evaluated as |N|^2-style Boolean matrix products (Valiant's view):
// for every non-preterminal A,
//     P_A[i][j] = Σ_{A->BC} Σ_r T_B[i][r] · T_C[r][j]   (integer, exact: ≤ |rules|·n < 2^31)
//     T_k,A[i][j] = T_{k-1},A[i][j] ∨ (P_A[i][j] > 0)        (N1·N2 per rule, ∪ over r)
// Operands are 0/1 bytes (T8 = row-major copy of T_B, T8T = transposed copy of T_C, both
// K-major for the UMMA), staged by TMA into 128B-swizzled shared memory; the s32
// accumulator lives in TMEM (128 lanes x 256 columns); the epilogue thresholds it to bits,
// ORs the old bits, writes T_k into the other bit-matrix buffer and counts new cells.
// Empty 128x128 operand tiles are skipped (tile-occupancy "skip list").
//
// Roles per CTA (persistent over output tiles (A, I, J), 128 x 256 each):
//   warp 0 : TMA producer (one elected lane)      -> full[s]
//   warp 1 : TMEM allocator + MMA issuer (one lane) -> empty[s], tmem_full
//   warps 2-5 : epilogue (TMEM -> registers -> bits)   -> tmem_empty
#include <cuda.h>
#include <cudaTypedefs.h>

#include "cfpq_internal.cuh"

namespace cfpq {

constexpr int kTM = 128;                 // UMMA M (rows of the output tile)
constexpr int kTN = 256;                 // UMMA N (columns of the output tile)
constexpr int kTK = 128;                 // K bytes per pipeline stage (one 128B swizzle row)
constexpr int kUK = 32;                  // K per tcgen05.mma kind::i8
constexpr int kStages = 4;
constexpr int kABytes = kTM * kTK;       // 16 KiB
constexpr int kBBytes = kTN * kTK;       // 32 KiB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kDenseThreads = 192;       // 6 warps
constexpr int kTmemCols = 512;          // two 256-column s32 accumulators

struct DenseRule {   // A -> B C, operand slots into the packed arrays
    int32_t A, B, C, pad;
};

struct DenseParams {
    int32_t n, np;                 // nodes, padded to a multiple of 256
    int64_t Wp;                    // words per bit-matrix row
    int32_t n_out;                 // non-preterminal NTs (outputs)
    const int32_t* out_nt;         // [n_out] NT ids
    const int32_t* rule_ptr;       // [n_out+1] rules of each output NT
    const DenseRule* rules;        // B, C = NT ids
    const uint32_t* const* T;      // [n_nt] current bit matrices (T_{k-1})
    uint32_t* const* Tn;           // [n_nt] next bit matrices (T_k); only outputs
    const uint8_t* occ;            // [n_nt][nt_tiles][nt_tiles] 128x128 tile occupancy
    int32_t nt_tiles;              // np / 128
    unsigned long long* new_cells; // [n_nt + 1] new cells per NT, [n_nt] = total
    int32_t n_nt;
    int32_t i_lo, i_hi;            // row-tile range of this rank (row-block sharding)
    int32_t j_lo, j_hi;            // column-tile range (256-column tiles; 2-D block sharding)
};

// ------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase: a tight try_wait loop in PTX.  (A C++ loop, or a poll counter for a
// watchdog, costs ~15% on config S: the four epilogue warps spinning on the accumulator
// barrier steal issue slots from the producer and MMA warps.)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
// Multicast variant: the box lands at the same CTA-relative offset in every CTA of
// cta_mask and completes bytes on each one's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               uint16_t cta_mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(cta_mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// kind::mxf4 (MXFP4: e2m1 operands packed two per byte, one ue8m0 scale per 32 K
// elements), block-scaled MMA M=128, N=256, K=64.  Scale factors are read from TMEM.
__device__ __forceinline__ void umma_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate, uint32_t tmem_sfa, uint32_t tmem_sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb));
}
// Fill 32 TMEM columns of this warp's 32 lanes with one 32-bit value.
__device__ __forceinline__ void tmem_fill32(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(v)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// Arrive on the mbarrier at this offset in every CTA of cta_mask once the MMAs complete.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major operand tile in 128B-swizzled shared memory (rows of 128 bytes, 8-row atoms
// 1024 B apart): start>>4, LBO = 1 (unused for swizzled K-major), SBO = 1024>>4,
// version 1 (sm_100), layout SWIZZLE_128B = 2.
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// kind::i8 instruction descriptor: D s32, A/B unsigned 8-bit, both K-major, M=128, N=256.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kind::mxf4 block-scaled instruction descriptor: A/B e2m1 (MXF4 format 1), K-major,
// scale format ue8m0 (bit 23), N>>3 at bit 17, M>>4 at bit 24, dense K = 64, scale ids 0.
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
constexpr uint32_t kSfOne = 0x7F7F7F7Fu;   // four ue8m0 scale bytes of 2^0 = 1.0

// ------------------------------------------------------------------------------------------
// Pack: bits -> 0/1 bytes (row-major T8 and transposed T8T) + 128x128 tile occupancy.
// One CTA (256 threads) per 128x128 tile of one NT.
// ------------------------------------------------------------------------------------------
// kF4: e2m1 nibbles instead of bytes (1.0 = 0x2, two elements per byte, element 2b in the
// low nibble of byte b); row length np/2 bytes.  A and B use the same K order, so the dot
// products are those of the byte packs.
//
// One CTA of 128 threads per 128x128 tile: thread t holds the 128 bits of tile row t (one
// 16-byte load).  Row-major pack: each thread expands its own bits.  Transposed pack: one
// warp ballot per column gives that column's 32 row bits of the warp's 32 rows, expanded
// by lane (column mod 32) — no shared-memory transpose.
__device__ __forceinline__ uint32_t spread8_nib(uint32_t x) {   // 8 bits -> 8 nibbles of value 0x2
    x &= 0xFFu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = (x | (x << 3)) & 0x11111111u;
    return x << 1;
}
__device__ __forceinline__ uint32_t spread4_byte(uint32_t x) {   // 4 bits -> 4 bytes of value 1
    return ((x & 0xFu) * 0x00204081u) & 0x01010101u;
}

template <bool kF4>
__global__ void __launch_bounds__(128) pack_kernel(const uint32_t* __restrict__ T, int32_t n, int64_t Wp, int32_t np,
                                                   uint8_t* T8, uint8_t* T8T, uint8_t* occ, int32_t nt_tiles) {
    // both packs of the tile are built in shared memory, then copied out with consecutive
    // lanes on consecutive 16-byte pieces of the same output rows (coalesced stores)
    constexpr int kRB = kF4 ? kTM / 2 : kTM;   // bytes of one packed tile row (64 fp4, 128 int8)
    __shared__ __align__(16) uint8_t s_rm[kTM * kRB];   // row-major pack of the tile
    __shared__ __align__(16) uint8_t s_tr[kTM * kRB];   // transposed pack of the tile
    __shared__ int any;
    const int tI = blockIdx.y, tK = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) any = 0;
    const int row = tI * kTM + t;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < n && (int64_t)tK * kTM < n) v = __ldg(reinterpret_cast<const uint4*>(T + (size_t)row * Wp) + tK);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    __syncthreads();
    if (__any_sync(0xffffffffu, (v.x | v.y | v.z | v.w) != 0) && lane == 0) any = 1;
    const int64_t rb = kF4 ? np / 2 : np;   // bytes per packed row in HBM
    if (T8) {
        uint4* dst = reinterpret_cast<uint4*>(s_rm + t * kRB);
        if (kF4) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(spread8_nib(w[q]), spread8_nib(w[q] >> 8), spread8_nib(w[q] >> 16),
                                    spread8_nib(w[q] >> 24));
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t x = w[q >> 1] >> ((q & 1) * 16);
                dst[q] = make_uint4(spread4_byte(x), spread4_byte(x >> 4), spread4_byte(x >> 8), spread4_byte(x >> 12));
            }
        }
    }
    if (T8T) {
        // column c = 32g + j: one ballot gives the warp's 32 row bits; lane j keeps its column
#pragma unroll
        for (int g = 0; g < kTM / 32; ++g) {
            uint32_t mine = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t m = __ballot_sync(0xffffffffu, (w[g] >> j) & 1u);
                if (lane == j) mine = m;
            }
            uint8_t* d = s_tr + (32 * g + lane) * kRB + (32 * warp) / (kF4 ? 2 : 1);
            if (kF4) {
                *reinterpret_cast<uint4*>(d) =
                    make_uint4(spread8_nib(mine), spread8_nib(mine >> 8), spread8_nib(mine >> 16), spread8_nib(mine >> 24));
            } else {
                uint4* d4 = reinterpret_cast<uint4*>(d);
                d4[0] = make_uint4(spread4_byte(mine), spread4_byte(mine >> 4), spread4_byte(mine >> 8),
                                   spread4_byte(mine >> 12));
                d4[1] = make_uint4(spread4_byte(mine >> 16), spread4_byte(mine >> 20), spread4_byte(mine >> 24),
                                   spread4_byte(mine >> 28));
            }
        }
    }
    __syncthreads();
    // copy out: kRB/16 pieces per row, consecutive threads on consecutive pieces
    constexpr int kPieces = kTM * kRB / 16;
    const size_t col_byte = (size_t)tK * kRB;
    const size_t tcol_byte = (size_t)tI * kRB;
    for (int e = t; e < kPieces; e += 128) {
        const int r = e / (kRB / 16), pc = e % (kRB / 16);
        if (T8)
            *reinterpret_cast<uint4*>(T8 + (size_t)(tI * kTM + r) * rb + col_byte + pc * 16) =
                reinterpret_cast<const uint4*>(s_rm + r * kRB)[pc];
        if (T8T)
            *reinterpret_cast<uint4*>(T8T + (size_t)(tK * kTM + r) * rb + tcol_byte + pc * 16) =
                reinterpret_cast<const uint4*>(s_tr + r * kRB)[pc];
    }
    if (t == 0 && occ) occ[(size_t)tI * nt_tiles + tK] = any ? 1 : 0;
}

// ------------------------------------------------------------------------------------------
// The tcgen05 product kernel
// ------------------------------------------------------------------------------------------
struct TileIter {   // walks the (A, I, J) output tiles of this CTA
    int32_t tiles_per_nt, n_i, n_j;
};

__device__ __forceinline__ bool kblock_live(const DenseParams& p, const DenseRule& r, int I, int J, int K) {
    const size_t tt = (size_t)p.nt_tiles * p.nt_tiles;
    const uint8_t* oB = p.occ + (size_t)r.B * tt;
    const uint8_t* oC = p.occ + (size_t)r.C * tt;
    if (!__ldg(oB + (size_t)I * p.nt_tiles + K)) return false;
    // B operand = T_C rows K-block, columns J*256 .. +255 = two 128x128 tiles of T_C
    return __ldg(oC + (size_t)K * p.nt_tiles + 2 * J) || __ldg(oC + (size_t)K * p.nt_tiles + 2 * J + 1);
}

// K block live for any of the kCl row tiles I0 .. I0+kCl-1 that exist (< i_hi).  kF4: a K
// block is 256 elements deep (128 bytes of nibbles) = 128-tiles 2K and 2K+1.
template <int kCl, bool kF4 = false>
__device__ __forceinline__ bool kblock_live_group(const DenseParams& p, const DenseRule& r, int I0, int J, int K) {
    bool live = false;
#pragma unroll
    for (int c = 0; c < kCl; ++c)
        if (I0 + c < p.i_hi) {
            if (kF4) live |= kblock_live(p, r, I0 + c, J, 2 * K) || kblock_live(p, r, I0 + c, J, 2 * K + 1);
            else live |= kblock_live(p, r, I0 + c, J, K);
        }
    return live;
}

// Live K blocks K0 .. K0+31 of (rule, row tile(s) I0, column tile J) as a bit mask: every lane
// checks one K block (its occupancy loads in parallel with the other lanes'), one ballot.
// The whole warp must call it.
template <int kCl, bool kF4>
__device__ __forceinline__ uint32_t live_mask32(const DenseParams& p, const DenseRule& r, int I0, int J, int K0,
                                                int n_k) {
    const int K = K0 + (int)(threadIdx.x & 31);
    const bool lv = K < n_k && kblock_live_group<kCl, kF4>(p, r, I0, J, K);
    return __ballot_sync(0xffffffffu, lv);
}

// Output tile t of this rank -> (output o, row tile I, column tile J).  Tiles of one output
// are walked in groups of kGroup row tiles, columns outer: a wave of ~148 CTAs then covers
// a kGroup x ~18 patch whose operand blocks (A: kGroup*128 rows, B: ~18*256 rows of the
// packs) fit in L2 together, instead of a 2-3 x 64 strip that streams all of B per wave.
constexpr int kGroup = 8;
__device__ __forceinline__ void tile_coords(const DenseParams& p, int t, int tiles_per_nt, int n_i, int n_j, int& o,
                                            int& I, int& J) {
    o = t / tiles_per_nt;
    const int rem = t - o * tiles_per_nt;
    const int g = rem / (kGroup * n_j);
    const int within = rem - g * (kGroup * n_j);
    const int rows_g = min(kGroup, n_i - g * kGroup);
    I = g * kGroup + within % rows_g;   // relative to the rank's first (pair of) row tile(s)
    J = p.j_lo + within / rows_g;        // absolute column tile
}

// kCl = 2: CTA pairs (thread-block clusters of 2) compute row tiles I0 and I0+1 of the same
// column tile J in lockstep over the same K blocks and share the B tile: each CTA loads one
// 128-row half and multicasts it into both CTAs' stage (half the B traffic from L2), and
// every MMA commit arrives on both CTAs' empty barrier (a stage is refilled only when both
// consumed it).  tmB's box is then 128 rows.
//
// kF4 (kind::mxf4, unit scales): operands are e2m1 nibble packs (K block = 256 elements in
// the same 128-byte swizzled rows), the f32 accumulator uses TMEM columns 0..255 (one
// accumulator stage) and columns 256..319 hold the scale factors, all 1.0 (ue8m0 0x7F).
// Every product term is 1.0 x 1.0 x 1 x 1 >= 0, so a sum is > 0 iff some term is, and the
// threshold is exact at any magnitude (and the sums are exact integers below 2^24).
template <int kCl, bool kF4 = false>
__global__ void __launch_bounds__(kDenseThreads, 1)
    dense_kernel(DenseParams p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const int64_t* __restrict__ mapA_row, const int64_t* __restrict__ mapB_row) {
    // mapA_row[X] = first row of NT X inside the stacked T8 tensor (tmA), mapB_row likewise
    // for the stacked T8T tensor (tmB); -1 if X is not packed.
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kKB = kTK, S_ = kStages, AB_ = kABytes, BB_ = kBBytes, SB_ = kStageBytes;
    uint8_t* sA = smem;                                  // [S_][AB_]
    uint8_t* sB = smem + S_ * AB_;                       // [S_][BB_]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_ * SB_);
    uint64_t* empty = full + S_;
    uint64_t* tmem_full = empty + S_;              // [2] accumulator stages (double-buffered TMEM)
    uint64_t* tmem_empty = tmem_full + 2;          // [2]
    uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_j = p.j_hi - p.j_lo;
    const int n_i = (p.i_hi - p.i_lo + kCl - 1) / kCl;   // (pairs of) row tiles
    const int tiles_per_nt = n_i * n_j;
    const int total_tiles = tiles_per_nt * p.n_out;
    const int n_k = kF4 ? p.np / (2 * kKB) : p.np / kKB;
    constexpr int kAcc = kF4 ? 1 : 2;   // accumulator stages in TMEM
    const uint32_t crank = kCl == 2 ? cluster_ctarank() : 0u;
    const int unit = (int)blockIdx.x / kCl, n_units = (int)gridDim.x / kCl;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S_; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCl);   // one MMA commit per CTA of the cluster
        }
        for (int a = 0; a < kAcc; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    if (warp == 1) tmem_alloc(tmem_base_smem, kTmemCols);
    tc_fence_before();
    if (kCl == 2) cluster_sync_all();   // barrier inits visible to the peer before its multicasts
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_smem;
    if (kF4) {
        // scale factors = 1.0 in columns 256..319 of all 128 lanes (epilogue warps own the
        // lane quarters), visible to the MMA issuer after the barrier
        if (warp >= 2) {
            const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
            tmem_fill32(tmem_base + lane_base + 256u, kSfOne);
            tmem_fill32(tmem_base + lane_base + 288u, kSfOne);
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }

    if (warp == 0) {
        // ------------------------------- TMA producer -------------------------------
        // the warp computes the skip list 32 K blocks at a time; lane 0 issues the loads
        int stage = 0;
        uint32_t phase = 0;
        for (int t = unit; t < total_tiles; t += n_units) {
            int o, I2, J;
            tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
            const int I0 = p.i_lo + I2 * kCl, I = I0 + (int)crank;
            for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1]; ++q) {
                const DenseRule r = p.rules[q];
                const int64_t arow = __ldg(mapA_row + r.B) + (int64_t)I * kTM;
                const int64_t brow = __ldg(mapB_row + r.C) + (int64_t)J * kTN;
                for (int K0 = 0; K0 < n_k; K0 += 32) {
                    uint32_t m = live_mask32<kCl, kF4>(p, r, I0, J, K0, n_k);
                    if (lane == 0) {
                        while (m) {
                            const int K = K0 + __ffs(m) - 1;
                            m &= m - 1u;
                            mbar_wait(&empty[stage], phase ^ 1);
                            mbar_expect_tx(&full[stage], SB_);
                            tma_load_2d(sA + stage * AB_, &tmA, &full[stage], K * kKB, (int)arow);
                            if (kCl == 1)
                                tma_load_2d(sB + stage * BB_, &tmB, &full[stage], K * kKB, (int)brow);
                            else
                                tma_load_2d_mc(sB + stage * BB_ + crank * (BB_ / 2), &tmB, &full[stage], K * kKB,
                                               (int)(brow + crank * (kTN / 2)), (uint16_t)0x3);
                            if (++stage == S_) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------- MMA issuer -------------------------------
        const uint32_t idesc = kF4 ? idesc_mxf4(kTM, kTN) : idesc_i8(kTM, kTN);
        const uint32_t tsfa = tmem_base + 256u, tsfb = tmem_base + 288u;
        int stage = 0;
        uint32_t phase = 0;
        int as = 0;              // accumulator stage of this tile
        uint32_t tphase = 0;     // phase of the stage's barriers
        for (int t = unit; t < total_tiles; t += n_units) {
            int o, I2, J;
            tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
            const int I0 = p.i_lo + I2 * kCl;
            const uint32_t tmem_acc = tmem_base + (uint32_t)(as * 256);
            // the epilogue must have drained this accumulator (tile t-2)
            mbar_wait(&tmem_empty[as], tphase ^ 1);
            tc_fence_after();
            uint32_t acc = 0;
            unsigned long long kb_issued = 0;
            for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1]; ++q) {
                const DenseRule r = p.rules[q];
                for (int K0 = 0; K0 < n_k; K0 += 32) {
                uint32_t m = live_mask32<kCl, kF4>(p, r, I0, J, K0, n_k);
                while (m) {
                    m &= m - 1u;
                    kb_issued += (kTN / 32) * (kF4 ? 2 : 1);   // in 128 x 32 x 128 units of MMA work
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * AB_);
                        const uint32_t b0 = smem_u32(sB + stage * BB_);
#pragma unroll
                        for (int kk = 0; kk < kKB / kUK; ++kk) {
                            // 32 bytes of K per instruction: 32 int8 or 64 e2m1 elements
                            const uint64_t ad = kmajor_sw128_desc(a0 + kk * kUK), bd = kmajor_sw128_desc(b0 + kk * kUK);
                            if (kF4)
                                umma_mxf4(tmem_acc, ad, bd, idesc, acc, tsfa, tsfb);
                            else
                                umma_i8(tmem_acc, ad, bd, idesc, acc);
                            acc = 1;
                        }
                        // frees the smem stage (in both CTAs of a pair) when these MMAs finish
                        if (kCl == 1) umma_commit(&empty[stage]);
                        else umma_commit_mc(&empty[stage], (uint16_t)0x3);
                    }
                    __syncwarp();
                    if (++stage == S_) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                }
            }
            if (lane == 0) {
                if (kb_issued) atomicAdd(p.new_cells + p.n_nt + 1, kb_issued);
                if (acc) umma_commit(&tmem_full[as]);   // arrives when all MMAs of the tile completed
                else mbar_arrive(&tmem_full[as]);       // no live K block: the epilogue uses zeros
            }
            __syncwarp();
            if (++as == kAcc) {
                as = 0;
                tphase ^= 1;
            }
        }
    } else {
        // ------------------------------- epilogue (warps 2..5) -------------------------------
        const int quarter = warp & 3;            // TMEM lanes 32*quarter .. +31 are this warp's
        int as = 0;
        uint32_t tphase = 0;
        unsigned long long my_new = 0;
        for (int t = unit; t < total_tiles; t += n_units) {
            int o, I2, J;
            tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
            const int I0 = p.i_lo + I2 * kCl, I = I0 + (int)crank;
            const bool mine = I < p.i_hi;   // the second tile of an odd last pair does not exist
            const int A = p.out_nt[o];
            bool live = false;   // the pair issued MMAs for this tile (else TMEM holds no result)
            for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1] && !live; ++q)
                for (int K0 = 0; K0 < n_k && !live; K0 += 32) live = live_mask32<kCl, kF4>(p, p.rules[q], I0, J, K0, n_k) != 0;
            // this row's 8 old words (32 contiguous bytes of T_{k-1}) load while the MMAs run
            const int row = I * kTM + quarter * 32 + lane;
            const bool wr = mine && row < p.n;
            uint4 o0 = make_uint4(0, 0, 0, 0), o1 = o0;
            if (wr) {
                const uint4* src = reinterpret_cast<const uint4*>(p.T[A] + (size_t)row * p.Wp + (size_t)J * (kTN / 32));
                o0 = __ldg(src);
                o1 = __ldg(src + 1);
            }
            mbar_wait(&tmem_full[as], tphase);
            tc_fence_after();
            uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (live) {
#pragma unroll 1
                for (int c = 0; c < kTN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(as * 256 + c * 32), v);
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 32; ++b) word |= (v[b] != 0u ? 1u : 0u) << b;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (q == c) w[q] = word;
                }
            }
            // the accumulator is in registers: hand TMEM back to the MMA issuer before the stores
            tc_fence_before();
            mbar_arrive(&tmem_empty[as]);
            if (++as == kAcc) {
                as = 0;
                tphase ^= 1;
            }
            unsigned long long cnt = 0;
            if (wr) {
                const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
                uint32_t nw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    nw[q] = old[q] | w[q];
                    cnt += __popc(w[q] & ~old[q]);
                }
                uint4* dst = reinterpret_cast<uint4*>(p.Tn[A] + (size_t)row * p.Wp + (size_t)J * (kTN / 32));
                dst[0] = make_uint4(nw[0], nw[1], nw[2], nw[3]);
                dst[1] = make_uint4(nw[4], nw[5], nw[6], nw[7]);
            }
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
            if (lane == 0 && cnt) atomicAdd(p.new_cells + A, cnt);
            my_new += cnt;
        }
        if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
    }
    tc_fence_before();
    // a CTA may not leave while its peer can still multicast into it or arrive on its barriers
    if (kCl == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

// ------------------------------------------------------------------------------------------
// 2-SM variant (cta_group::2): a CTA pair computes a 256 x 256 output tile with M=256 UMMAs
// issued by the even CTA.  Each CTA stages its own 128 rows of A and its 128-row half of B
// (32 KiB per K block instead of 48: a third less L2->SMEM traffic per MMA and 6 stages of
// buffering instead of 4); the TMA of both CTAs completes on the leader's full barrier, the
// leader's commits arrive on both CTAs' empty / accumulator barriers (multicast), and each
// CTA's epilogue reads its own 128 TMEM lanes (rows) x 256 columns and arrives on the
// leader's accumulator-empty barrier.  Same tile order, skip list and epilogue as above.
// ------------------------------------------------------------------------------------------
constexpr int kStages2 = 6;
constexpr int kBHalf = (kTN / 2) * kTK;             // 16 KiB: this CTA's half of the B tile
constexpr int kStage2Bytes = kABytes + kBHalf;       // 32 KiB

__device__ __forceinline__ uint32_t mapa_cta(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_remote(uint32_t cluster_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
                 "r"(bytes)
                 : "memory");
}
// TMA into this CTA's smem, completing bytes on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma2_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate, uint32_t tmem_sfa, uint32_t tmem_sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb));
}
__device__ __forceinline__ void umma2_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}

size_t dense2_smem_bytes() { return (size_t)kStages2 * kStage2Bytes + 1024 + 256; }

template <bool kF4>
__global__ void __launch_bounds__(kDenseThreads, 1)
    dense2sm_kernel(DenseParams p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                    const int64_t* __restrict__ mapA_row, const int64_t* __restrict__ mapB_row) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                  // [kStages2][kABytes]
    uint8_t* sB = smem + kStages2 * kABytes;             // [kStages2][kBHalf]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStage2Bytes);
    uint64_t* empty = full + kStages2;
    uint64_t* tmem_full = empty + kStages2;        // [kAcc]
    uint64_t* tmem_empty = tmem_full + 2;          // [kAcc] (leader's is the one used)
    uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    constexpr int kAcc = kF4 ? 1 : 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_j = p.j_hi - p.j_lo;
    const int n_i = (p.i_hi - p.i_lo + 1) / 2;        // pairs of row tiles
    const int tiles_per_nt = n_i * n_j;
    const int total_tiles = tiles_per_nt * p.n_out;
    const int n_k = kF4 ? p.np / (2 * kTK) : p.np / kTK;
    const uint32_t crank = cluster_ctarank();
    const bool leader = crank == 0;
    const int unit = (int)blockIdx.x / 2, n_units = (int)gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full[s], 1);    // the leader's producer arrives with both CTAs' bytes
            mbar_init(&empty[s], 1);   // the leader's MMA commit (multicast)
        }
        for (int a = 0; a < kAcc; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 8);   // one per epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmBh) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_smem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_smem;
    if (kF4) {
        if (warp >= 2) {
            const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
            tmem_fill32(tmem_base + lane_base + 256u, kSfOne);
            tmem_fill32(tmem_base + lane_base + 288u, kSfOne);
        }
        tc_fence_before();
        cluster_sync_all();   // both CTAs' scale factors before the first pair MMA
        tc_fence_after();
    }

    if (warp == 0) {
        // ------------------------------- TMA producer (both CTAs) -------------------------------
        {
            const uint32_t full0 = mapa_cta(smem_u32(&full[0]), 0);   // leader's full barriers
            int stage = 0;
            uint32_t phase = 0;
            for (int t = unit; t < total_tiles; t += n_units) {
                int o, I2, J;
                tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
                const int I0 = p.i_lo + I2 * 2, I = I0 + (int)crank;
                for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1]; ++q) {
                    const DenseRule r = p.rules[q];
                    const int64_t arow = __ldg(mapA_row + r.B) + (int64_t)I * kTM;
                    const int64_t brow = __ldg(mapB_row + r.C) + (int64_t)J * kTN + (int64_t)crank * (kTN / 2);
                    for (int K0 = 0; K0 < n_k; K0 += 32) {
                    uint32_t m = live_mask32<2, kF4>(p, r, I0, J, K0, n_k);
                    if (lane == 0)
                    while (m) {
                        const int K = K0 + __ffs(m) - 1;
                        m &= m - 1u;
                        mbar_wait(&empty[stage], phase ^ 1);
                        const uint32_t fb = full0 + (uint32_t)(stage * 8);
                        // no cluster-scope arrive from the peer: its TMA bytes complete on the
                        // leader's barrier, whose one arrival expects both CTAs' bytes (the
                        // transaction count may go transiently negative)
                        if (leader) mbar_expect_tx(&full[stage], 2 * kStage2Bytes);
                        tma_load_2d_pair(sA + stage * kABytes, &tmA, fb, K * kTK, (int)arow);
                        tma_load_2d_pair(sB + stage * kBHalf, &tmBh, fb, K * kTK, (int)brow);
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    __syncwarp();
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------- MMA issuer (leader CTA only) -------------------------------
        if (leader) {
            const uint32_t idesc = kF4 ? idesc_mxf4(2 * kTM, kTN) : idesc_i8(2 * kTM, kTN);
            const uint32_t tsfa = tmem_base + 256u, tsfb = tmem_base + 288u;
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t tphase = 0;
            for (int t = unit; t < total_tiles; t += n_units) {
                int o, I2, J;
                tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
                const int I0 = p.i_lo + I2 * 2;
                const uint32_t tmem_acc = tmem_base + (uint32_t)(as * 256);
                mbar_wait(&tmem_empty[as], tphase ^ 1);
                tc_fence_after();
                uint32_t acc = 0;
                unsigned long long kb_issued = 0;
                for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1]; ++q) {
                    const DenseRule r = p.rules[q];
                    for (int K0 = 0; K0 < n_k; K0 += 32) {
                    uint32_t m = live_mask32<2, kF4>(p, r, I0, J, K0, n_k);
                    while (m) {
                        m &= m - 1u;
                        kb_issued += 2 * (kTN / 32) * (kF4 ? 2 : 1);   // 128x32x128 units: two row tiles, fp4 twice as deep
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        if (lane == 0) {
                            const uint32_t a0 = smem_u32(sA + stage * kABytes);
                            const uint32_t b0 = smem_u32(sB + stage * kBHalf);
#pragma unroll
                            for (int kk = 0; kk < kTK / kUK; ++kk) {
                                if (kF4)
                                    umma2_mxf4(tmem_acc, kmajor_sw128_desc(a0 + kk * kUK), kmajor_sw128_desc(b0 + kk * kUK),
                                               idesc, acc, tsfa, tsfb);
                                else
                                    umma2_i8(tmem_acc, kmajor_sw128_desc(a0 + kk * kUK), kmajor_sw128_desc(b0 + kk * kUK),
                                             idesc, acc);
                                acc = 1;
                            }
                            umma2_commit_mc(&empty[stage], (uint16_t)0x3);
                        }
                        __syncwarp();
                        if (++stage == kStages2) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    }
                }
                if (lane == 0) {
                    if (kb_issued) atomicAdd(p.new_cells + p.n_nt + 1, kb_issued);
                    if (acc) {
                        umma2_commit_mc(&tmem_full[as], (uint16_t)0x3);
                    } else {
                        // no live K block: both epilogues proceed on zeros
                        mbar_arrive(&tmem_full[as]);
                        mbar_arrive_remote(mapa_cta(smem_u32(&tmem_full[as]), 1));
                    }
                }
                __syncwarp();
                if (++as == kAcc) {
                    as = 0;
                    tphase ^= 1;
                }
            }
        }
    } else {
        // ------------------------------- epilogue (warps 2..5, both CTAs) -------------------------------
        const int quarter = warp & 3;
        int as = 0;
        uint32_t tphase = 0;
        unsigned long long my_new = 0;
        const uint32_t empty0 = mapa_cta(smem_u32(&tmem_empty[0]), 0);
        for (int t = unit; t < total_tiles; t += n_units) {
            int o, I2, J;
            tile_coords(p, t, tiles_per_nt, n_i, n_j, o, I2, J);
            const int I0 = p.i_lo + I2 * 2, I = I0 + (int)crank;
            const bool mine = I < p.i_hi;
            const int A = p.out_nt[o];
            bool live = false;
            for (int q = p.rule_ptr[o]; q < p.rule_ptr[o + 1] && !live; ++q)
                for (int K0 = 0; K0 < n_k && !live; K0 += 32) live = live_mask32<2, kF4>(p, p.rules[q], I0, J, K0, n_k) != 0;
            const int row = I * kTM + quarter * 32 + lane;
            const bool wr = mine && row < p.n;
            uint4 o0 = make_uint4(0, 0, 0, 0), o1 = o0;
            if (wr) {
                const uint4* src = reinterpret_cast<const uint4*>(p.T[A] + (size_t)row * p.Wp + (size_t)J * (kTN / 32));
                o0 = __ldg(src);
                o1 = __ldg(src + 1);
            }
            mbar_wait(&tmem_full[as], tphase);
            tc_fence_after();
            uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (live) {
#pragma unroll 1
                for (int c = 0; c < kTN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(as * 256 + c * 32), v);
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 32; ++b) word |= (v[b] != 0u ? 1u : 0u) << b;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (q == c) w[q] = word;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(empty0 + (uint32_t)(as * 8));
            if (++as == kAcc) {
                as = 0;
                tphase ^= 1;
            }
            unsigned long long cnt = 0;
            if (wr) {
                const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
                uint32_t nw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    nw[q] = old[q] | w[q];
                    cnt += __popc(w[q] & ~old[q]);
                }
                uint4* dst = reinterpret_cast<uint4*>(p.Tn[A] + (size_t)row * p.Wp + (size_t)J * (kTN / 32));
                dst[0] = make_uint4(nw[0], nw[1], nw[2], nw[3]);
                dst[1] = make_uint4(nw[4], nw[5], nw[6], nw[7]);
            }
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
            if (lane == 0 && cnt) atomicAdd(p.new_cells + A, cnt);
            my_new += cnt;
        }
        if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
    }
    tc_fence_before();
    cluster_sync_all();   // all MMAs consumed, all epilogues done in both CTAs
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
}

// ------------------------------------------------------------------------------------------
// Bit-row path (CUDA cores, path_policy 3): Alg. 1 line 9 as written — every iteration the
// FULL Jacobi product T_{k-1} x T_{k-1} (not only Δ), over packed rows:
//   T_k,A[i] = T_{k-1},A[i] | OR_{A->BC} OR_{r : T_B[i][r]} T_C[r]
// Each rule is evaluated in the form its operands allow (preterminals are constant after
// seeding and have CSR rows):
//   L  B changes, C preterminal : scan the bit row T_B[i], scatter CSR_C(r) into row i
//   R  B preterminal, C changes : OR the bit rows T_C[r], r in CSR_B(i), into row i
//   V  both change              : OR the bit rows T_C[r], r a set bit of T_B[i], into row i
//   P  both preterminal         : CSR_B(i) x CSR_C(r); constant, so iteration 1 only
// Empty rows are skipped through per-row popcounts cnt[X][i] of the current T (grown in
// place by the merges: a count read during iteration k is >= that of T_{k-1}, and a row
// that gained bits only in T_k is still empty in the T_{k-1} buffer that is read).
// Merges are atomicOr into row i of T_k (after a plain-load pre-check); the bits an atomic
// flips are exactly the new cells: they are counted, added to cnt, and appended as
// (A, i, word, bits) to the word list Δ_k.  T_k is built in the buffer that held T_{k-2}:
// it starts as T_{k-2} | Δ_{k-1} (= T_{k-1}), a scatter of the word list instead of a
// copy of whole matrices (a full copy only if the list overflowed); at iteration 1 the
// zeroed buffer takes the seed cells from the log.
// ------------------------------------------------------------------------------------------
constexpr int kRowThreads = 256;
constexpr int kChunk = 128;     // set bits of T_B[i] per V chunk
constexpr int kChunkR = 32;     // CSR_B(i) entries per R chunk
constexpr int kChunkL = 64;     // set bits of T_B[i] per L chunk
constexpr int kRowMaxV4 = 8;    // uint4 accumulators per thread: rows up to 8*4*32*256 = 262144 bits
constexpr int kScanBatch = 4;   // 128-bit loads per lane in flight in the L-form row scan


struct RowChunk {
    int32_t rule;   // index into rules (output o implied)
    int32_t row;
    int32_t first;  // V: rank of the first set bit; R: first CSR_B(i) entry
    int32_t count;
};

// Δ_k word list and counters of the bit-row path
struct RowsCtx {
    const NTInfo* nt;                  // is_const, csr_ptr per NT
    const int32_t* adj_idx;            // CSR index array
    uint32_t* cnt;                     // [n_nt][n] popcount of row i of the current T_X
    uint4* dlist;                      // {A, i, word, bits}
    unsigned long long dlist_cap;
    unsigned long long* rc;            // [0] R chunks, [1] dlist entries, [2] dlist overflowed (sticky),
                                       // [3] V chunks, [4] L/P tasks
    int32_t first;                     // iteration 1 (both-preterminal rules evaluated)
    int32_t n_rules;
    int32_t row_lo, row_hi;            // rows this shard derives (row-block sharding; [0, n) else)
    const int32_t* l_next;             // L-form rules sharing B: next rule of the group (-1 = last);
                                       // l_next[q] = -2 marks a rule that is not a group leader
    unsigned long long chunk_cap;      // capacity of each chunk list (the products clamp to it;
                                       // the host re-runs the shard when a list overflowed)
    int32_t push;                      // form R by input row: chunks of CSC_B(r) (rows_rpush_kernel)
    // compact mode (unsharded runs without V rules): the plan lists whole operand rows with an
    // output offset; rows_compact_kernel streams them into entry lists (L: set bits of T_B[i],
    // R: non-zero words of T_C[r]); rows_lmerge / rows_rmerge merge the entries
    int32_t compact;
    uint4* elist;                      // [2 * ecap]: L entries, then R entries
    unsigned long long ecap;
    // pipelined iterations: a device flag set by rows_end_kernel (fixpoint, cap or a list that
    // ran out); every kernel of a later, speculatively enqueued iteration then does nothing
    const int* stop;
};

#define ROWS_GATE(c)                                                  \
    do {                                                              \
        if ((c).stop && *(volatile const int*)(c).stop) return;       \
    } while (0)

enum : int { RF_NONE = 0, RF_L = 1, RF_R = 2, RF_V = 3, RF_P = 4 };

// Next rule of an L-form group from RowsCtx::l_next (-1: none).
__device__ __forceinline__ int rows_l_follow(int v) { return v >= 0 ? v : (v <= -3 ? -(v + 3) : -1); }

__device__ __forceinline__ int row_form(const RowsCtx& c, const DenseRule& r) {
    const bool bc = c.nt[r.B].is_const, cc = c.nt[r.C].is_const;
    if (!bc && cc) return RF_L;
    if (bc && !cc) return RF_R;
    if (!bc && !cc) return RF_V;
    return c.first ? RF_P : RF_NONE;
}

// OR `bits` into word w of row i of T_k,A; record what flips.  Warp-aggregated list append.
__device__ __forceinline__ void rows_merge(const DenseParams& p, const RowsCtx& c, int A, int i, int64_t w,
                                           uint32_t bits, unsigned long long& my_new) {
    CFPQ_DASSERT(A >= 0 && A < p.n_nt && i >= 0 && i < p.n && w >= 0 && w < p.Wp && p.Tn[A] != nullptr);
    uint32_t* addr = p.Tn[A] + (size_t)i * p.Wp + w;
    uint32_t fl = 0;
    if (bits & ~*addr) fl = bits & ~atomicOr(addr, bits);   // bits never clear: a stale load only costs the atomic
    const unsigned m = __activemask();
    const unsigned want = __ballot_sync(m, fl != 0);
    if (!fl) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(want) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(c.rc + 1, (unsigned long long)__popc(want));
    base = __shfl_sync(want, base, leader);
    const unsigned long long at = base + __popc(want & ((1u << lane) - 1u));
    if (at < c.dlist_cap) c.dlist[at] = make_uint4((uint32_t)A, (uint32_t)i, (uint32_t)w, fl);
    atomicAdd(c.cnt + (size_t)A * p.n + i, (uint32_t)__popc(fl));
    my_new += __popc(fl);
}

// Per-shard counter reset in one launch: chunk list R (rc[0]), optionally the Δ list length
// (rc[1]), lists V / L-P and the compact entry slots (rc[3..6]); rc[2] (sticky) is kept.
__global__ void rows_reset_kernel(unsigned long long* rc, int with_list, const int* stop) {
    if (stop && *(volatile const int*)stop) return;
    const int t = threadIdx.x;
    if (t == 0 || (t == 1 && with_list) || (t >= 3 && t <= 6)) rc[t] = 0ull;
}

// Iteration 1: the zeroed T_k buffers take T_0 (the seed cells of the outputs, from the
// log) and cnt[X][i] = |row i of T_0,X| for every NT.
__global__ void rows_seed_kernel(DenseParams p, RowsCtx c, const uint64_t* __restrict__ log, unsigned long long n_seeds) {
    ROWS_GATE(c);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_seeds;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const uint64_t cell = log[e];
        const uint32_t A = cell_nt(cell), i = cell_i(cell), j = cell_j(cell);
        CFPQ_DASSERT(A < (uint32_t)p.n_nt && i < (uint32_t)p.n && j < (uint32_t)p.n);
        atomicAdd(c.cnt + (size_t)A * p.n + i, 1u);
        if (p.Tn[A]) atomicOr(p.Tn[A] + (size_t)i * p.Wp + (j >> 5), 1u << (j & 31));
    }
}

// Iteration k > 1: T_k buffer (holding T_{k-2}) |= Δ_{k-1} words; after an overflowed list,
// copy T_{k-1} whole (and flag it for the host to grow the list).
__global__ void rows_delta_kernel(DenseParams p, RowsCtx c, int copy_whole) {
    ROWS_GATE(c);
    const unsigned long long m = c.rc[1];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t0 = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (!copy_whole && m <= c.dlist_cap) {   // the list of Δ_{k-1} is complete
        for (unsigned long long e = t0; e < m; e += stride) {
            const uint4 d = c.dlist[e];
            CFPQ_DASSERT(e < c.dlist_cap && d.x < (uint32_t)p.n_nt && d.y < (uint32_t)p.n && d.z < (uint32_t)p.Wp);
            atomicOr(p.Tn[d.x] + (size_t)d.y * p.Wp + d.z, d.w);
        }
        return;
    }
    const unsigned long long words4 = (unsigned long long)p.n * p.Wp / 4;
    for (int o = 0; o < p.n_out; ++o) {
        const int A = p.out_nt[o];
        const uint4* src = reinterpret_cast<const uint4*>(p.T[A]);
        uint4* dst = reinterpret_cast<uint4*>(p.Tn[A]);
        for (unsigned long long e = t0; e < words4; e += stride) dst[e] = src[e];
    }
}

// Work lists of the R and V forms: chunks of <= kChunkR CSR_B(i) entries (list R at
// chunks[0, rc[0])) / kChunk set bits of T_B[i] (list V at chunks[cap, cap + rc[3])) per
// (rule, row), warp-aggregated appends.
constexpr int kPlanRules = 64;   // rule forms cached in shared memory up to this many rules

__global__ void rows_plan_kernel(DenseParams p, RowsCtx c, RowChunk* chunks, unsigned long long cap) {
    ROWS_GATE(c);
    __shared__ int32_t s_form[kPlanRules], s_B[kPlanRules];
    __shared__ const int32_t* s_ptr[kPlanRules];
    __shared__ int32_t s_wsum[5][32];
    __shared__ unsigned long long s_base[5];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int32_t s_active[kPlanRules];   // rules with work this iteration (cached plans)
    __shared__ int32_t s_nact;
    const bool cached = c.n_rules <= kPlanRules;
    int n_task_rules = c.n_rules;
    if (cached) {
        for (int q = threadIdx.x; q < c.n_rules; q += blockDim.x) {
            const DenseRule r = p.rules[q];
            s_form[q] = row_form(c, r);
            s_B[q] = r.B;
            s_ptr[q] = c.nt[r.B].csr_ptr;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // skip rules without tasks: no form this iteration (both operands preterminal after
            // iteration 1) and L rules that follow their group's leader
            int na = 0;
            for (int q = 0; q < c.n_rules; ++q)
                if (s_form[q] != RF_NONE && !(s_form[q] == RF_L && c.l_next[q] < -1)) s_active[na++] = q;
            s_nact = na;
        }
        __syncthreads();
        n_task_rules = s_nact;
    }
    const int64_t tasks = (int64_t)n_task_rules * (c.row_hi - c.row_lo);   // this shard's rows only
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x; t0 < tasks; t0 += stride) {
        const int64_t t = t0 + threadIdx.x;
        int nch = 0, q = 0, i = 0, per = 1, len = 0, isv = 0, lp = 0, lpl = 0;
        if (t < tasks) {
            // row-major: the rules of one row are adjacent in every list, so a bit row read
            // for two rules (e.g. S5 -> S P_sc and S6 -> S P_t) is re-read from L2
            if (tasks < (1ll << 31)) {
                i = (int)((uint32_t)t / (uint32_t)n_task_rules);
                q = (int)((uint32_t)t - (uint32_t)i * (uint32_t)n_task_rules);
            } else {
                i = (int)(t / n_task_rules);
                q = (int)(t - (int64_t)i * n_task_rules);
            }
            if (cached) q = s_active[q];
            i += c.row_lo;
            DenseRule r;
            int f;
            const int32_t* bptr;
            if (cached) {
                f = s_form[q];
                r.B = s_B[q];
                bptr = s_ptr[q];
            } else {
                r = p.rules[q];
                f = row_form(c, r);
                bptr = c.nt[r.B].csr_ptr;
            }
            if (f == RF_R && c.compact) {
                // compact: one task per non-empty input row T_C[r] with output rows (CSC_B(r));
                // its entries (<= cnt non-zero words) get slots [off, off + cnt) of the R list
                const int32_t* cp = c.nt[r.B].csc_ptr;
                const uint32_t cc = c.cnt[(size_t)p.rules[q].C * p.n + i];
                if (cc && __ldg(cp + i + 1) > __ldg(cp + i)) {
                    len = (int)cc;
                    per = 1 << 30;   // one task
                }
            } else if (f == RF_L && c.compact) {
                // compact: one task per non-empty T_B[i] per group of L rules sharing B; its set
                // bits get slots [off, off + cnt) of the L list
                if (c.l_next[q] >= -1) {
                    len = (int)c.cnt[(size_t)r.B * p.n + i];
                    per = 1 << 30;
                    isv = 1;         // listed in the V slot (unused in compact mode)
                }
            } else if (f == RF_P && c.compact) {
                // compact, iteration 1: both operands preterminal — the set bits of T_B[i] (= CSR_B(i),
                // constant) listed like an L row; the merge applies this rule alone (not a group)
                len = (int)c.cnt[(size_t)r.B * p.n + i];
                per = 1 << 30;
                isv = 1;
            } else if (f == RF_R && c.push) {
                // push form: task row = input row r of T_C (non-empty), chunks of CSC_B(r)
                const int32_t* cp = c.nt[r.B].csc_ptr;
                len = c.cnt[(size_t)p.rules[q].C * p.n + i] ? __ldg(cp + i + 1) - __ldg(cp + i) : 0;
                per = kChunkR;
            } else if (f == RF_R) {
                const int32_t* ptr = bptr;
                len = __ldg(ptr + i + 1) - __ldg(ptr + i);
                per = kChunkR;
            } else if (f == RF_V) {
                len = (int)c.cnt[(size_t)r.B * p.n + i];
                per = kChunk;
                isv = 1;
            } else if (f == RF_L) {
                // chunks of <= kChunkL set bits of T_B[i] (hub rows over many warps); one task
                // per group of L rules with the same B (the leader scans the row once for all)
                if (c.l_next[q] >= -1) {   // a group leader
                    lp = (int)((c.cnt[(size_t)r.B * p.n + i] + kChunkL - 1) / kChunkL);
                    lpl = (int)c.cnt[(size_t)r.B * p.n + i];
                }
            } else if (f == RF_P) {
                const int32_t* ptr = bptr;
                lp = __ldg(ptr + i + 1) > __ldg(ptr + i);
            }
            nch = (len + per - 1) / per;
        }
        // three lists: 0 = R chunks (rc[0]), 1 = V chunks (rc[3]), 2 = L chunks / P tasks (rc[4]);
        // compact mode also sums the entry slots of its R tasks (rc[6]) and L tasks (rc[5]).
        // Warp inclusive scans, then one atomic per list per CTA (not per warp: the
        // counters are hot), bases handed back through shared memory
        const bool cpt = c.compact && nch == 1 && per == (1 << 30);
        const int cntv[5] = {isv ? 0 : nch, isv ? nch : 0, lp, cpt && !isv ? len : 0, cpt && isv ? len : 0};
        int incl[5];
#pragma unroll
        for (int l = 0; l < 5; ++l) {
            incl[l] = cntv[l];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(0xffffffffu, incl[l], o);
                if (lane >= o) incl[l] += v;
            }
            if (lane == 31) s_wsum[l][warp] = incl[l];
        }
        __syncthreads();
        if (threadIdx.x < 5) {
            const int l = threadIdx.x;
            unsigned long long tot = 0;
            for (int q2 = 0; q2 < (int)(blockDim.x >> 5); ++q2) tot += (unsigned long long)s_wsum[l][q2];
            const int ctr[5] = {0, 3, 4, 6, 5};
            s_base[l] = tot ? atomicAdd(c.rc + ctr[l], tot) : 0ull;
        }
        __syncthreads();
        unsigned long long ebase = 0;   // compact task: its first entry slot
        if (cpt) {
            const int l = isv ? 4 : 3;
            ebase = s_base[l];
            for (int q2 = 0; q2 < warp; ++q2) ebase += (unsigned long long)s_wsum[l][q2];
            ebase += (unsigned long long)(incl[l] - cntv[l]);
        }
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            unsigned long long at = s_base[l];
            for (int q2 = 0; q2 < warp; ++q2) at += (unsigned long long)s_wsum[l][q2];
            at += (unsigned long long)(incl[l] - cntv[l]);
            if (l < 2) {
                RowChunk* out = chunks + (l ? cap : 0);
                if (cpt) {
                    // first = the entry slot (< 2^31: the host caps the entry lists below it)
                    if (cntv[l] && at < cap) out[at] = RowChunk{q, i, (int32_t)ebase, len};
                    continue;
                }
                for (int h = 0; h < cntv[l]; ++h, ++at)
                    if (at < cap) out[at] = RowChunk{q, i, h * per, min(per, len - h * per)};
            } else {
                for (int h = 0; h < lp; ++h, ++at)
                    if (at < cap)
                        chunks[2 * cap + at] = RowChunk{q, i, h * kChunkL, lpl ? min(kChunkL, lpl - h * kChunkL) : 0};
            }
        }
        __syncthreads();   // s_wsum / s_base are rewritten by the next iteration
    }
}

// Form R, one warp per (chunk, row slice of 32 * NVW uint4): lane e holds CSR_B(i) entry
// e, the non-empty rows T_C[r] are ORed one after another with NVW 128-bit loads per lane
// in flight, then the non-zero words of the slice are merged.  No CTA barriers.
template <int NVW, int RU, int MINB>
__global__ void __launch_bounds__(256, MINB) rows_rgather_kernel(DenseParams p, RowsCtx c, const int32_t* __restrict__ rule_out,
                                                                 const RowChunk* __restrict__ chunks) {
    // RU rows of T_C in flight per step (RU x NVW 128-bit loads per lane issued before the
    // ORs): the R form is latency-bound on the load -> OR dependence of one row at a time
    const int lane = threadIdx.x & 31;
    const int64_t nv4 = ((p.n + 31) / 32 + 3) / 4;
    const int parts = (int)((nv4 + 32 * NVW - 1) / (32 * NVW));   // row slices of 32*NVW uint4
    const unsigned long long m = min(c.rc[0], c.chunk_cap) * (unsigned long long)parts;
    unsigned long long my_new = 0;
    for (unsigned long long ti = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5; ti < m;
         ti += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
        const unsigned long long ci = ti / parts;
        const int64_t vbase = (int64_t)(ti - ci * parts) * 32 * NVW;
        const RowChunk ch = chunks[ci];
        const DenseRule r = p.rules[ch.rule];
        int rr = 0;
        bool ok = false;
        if (lane < ch.count) {
            rr = __ldg(c.adj_idx + __ldg(c.nt[r.B].csr_ptr + ch.row) + ch.first + lane);
            ok = c.cnt[(size_t)r.C * p.n + rr] != 0;
        }
        unsigned todo = __ballot_sync(0xffffffffu, ok);
        if (!todo) continue;
        uint4 acc[NVW];
#pragma unroll
        for (int b = 0; b < NVW; ++b) acc[b] = make_uint4(0, 0, 0, 0);
        const uint4* TC = reinterpret_cast<const uint4*>(p.T[r.C]);
        const int64_t wp4 = p.Wp / 4;
        while (todo) {
            int rows_u[RU];
            bool have[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                have[u] = todo != 0u;   // warp-uniform
                const int src_lane = have[u] ? __ffs(todo) - 1 : 0;
                if (have[u]) todo &= todo - 1u;
                rows_u[u] = __shfl_sync(0xffffffffu, rr, src_lane);
            }
            uint4 x[RU][NVW];
#pragma unroll
            for (int u = 0; u < RU; ++u)
#pragma unroll
                for (int b = 0; b < NVW; ++b) {
                    const int64_t v = vbase + (int64_t)b * 32 + lane;
                    x[u][b] = have[u] && v < nv4 ? __ldg(TC + (size_t)rows_u[u] * wp4 + v) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
            for (int u = 0; u < RU; ++u)
#pragma unroll
                for (int b = 0; b < NVW; ++b) {
                    acc[b].x |= x[u][b].x;
                    acc[b].y |= x[u][b].y;
                    acc[b].z |= x[u][b].z;
                    acc[b].w |= x[u][b].w;
                }
        }
        const int A = rule_out[ch.rule];
#pragma unroll
        for (int b = 0; b < NVW; ++b) {
            const int64_t v = vbase + (int64_t)b * 32 + lane;
            const uint32_t a[4] = {acc[b].x, acc[b].y, acc[b].z, acc[b].w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (a[q]) rows_merge(p, c, A, ch.row, 4 * v + q, a[q], my_new);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// Form R by input row (push; unsharded runs): T_k[i] |= T_{k-1},C[r] for every i in CSC_B(r)
// — the same OR as the gather over CSR_B(i), but every non-empty row T_C[r] is streamed once
// per rule and iteration.  One warp per (chunk of <= kChunkR CSC_B(r) entries, row slice of
// 32 * NVW uint4): the slice and the chunk's output rows are loaded together, and the slice's
// non-zero words are merged into each output row.
template <int NVW, int MINB>
__global__ void __launch_bounds__(256, MINB) rows_rpush_kernel(DenseParams p, RowsCtx c, const int32_t* __restrict__ rule_out,
                                                               const RowChunk* __restrict__ chunks) {
    const int lane = threadIdx.x & 31;
    const int64_t nv4 = ((p.n + 31) / 32 + 3) / 4;
    const int parts = (int)((nv4 + 32 * NVW - 1) / (32 * NVW));
    const unsigned long long m = min(c.rc[0], c.chunk_cap) * (unsigned long long)parts;
    const int64_t wp4 = p.Wp / 4;
    unsigned long long my_new = 0;
    for (unsigned long long ti = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5; ti < m;
         ti += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
        const unsigned long long ci = ti / parts;
        const int64_t vbase = (int64_t)(ti - ci * parts) * 32 * NVW;
        const RowChunk ch = chunks[ci];
        const DenseRule r = p.rules[ch.rule];
        const uint4* row = reinterpret_cast<const uint4*>(p.T[r.C]) + (size_t)ch.row * wp4;
        uint4 x[NVW];
#pragma unroll
        for (int b = 0; b < NVW; ++b) {
            const int64_t v = vbase + (int64_t)b * 32 + lane;
            x[b] = v < nv4 ? __ldg(row + v) : make_uint4(0, 0, 0, 0);
        }
        CFPQ_DASSERT(ch.row >= 0 && ch.row < p.n && ch.count <= 32);
        const int ii = lane < ch.count ? __ldg(c.adj_idx + __ldg(c.nt[r.B].csc_ptr + ch.row) + ch.first + lane) : 0;
        bool nz = false;
#pragma unroll
        for (int b = 0; b < NVW; ++b) nz |= (x[b].x | x[b].y | x[b].z | x[b].w) != 0u;
        if (!__any_sync(0xffffffffu, nz)) continue;
        const int A = rule_out[ch.rule];
        for (int e = 0; e < ch.count; ++e) {
            const int i = __shfl_sync(0xffffffffu, ii, e);
#pragma unroll
            for (int b = 0; b < NVW; ++b) {
                const int64_t v = vbase + (int64_t)b * 32 + lane;
                const uint32_t a[4] = {x[b].x, x[b].y, x[b].z, x[b].w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (a[q]) rows_merge(p, c, A, i, 4 * v + q, a[q], my_new);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// ---- compact mode: stream whole operand rows into entry lists, then merge the entries ----
// The streaming pass reads each listed row once (16-byte loads, kCompactB per lane in flight)
// and is HBM-bound; the merges (adjacency lookups, pre-check, atomic) run as one thread per
// entry over the whole GPU instead of inside the warp that scanned the row.
constexpr int kCompactB = 4;

// MODE 0 (L): tasks = (leader rule, row i of T_B, slot, count) -> entries {rule, i, r, 1} for
// every set bit r of T_{k-1},B[i].  MODE 1 (R): tasks = (rule, row r of T_C, slot, count) ->
// entries {rule, r, word, bits} for every non-zero word.  Slots past the row's entries are
// written invalid (w = 0): count is the row's popcount in T_k, an upper bound.
template <int MODE>
__global__ void __launch_bounds__(256) rows_compact_kernel(DenseParams p, RowsCtx c, const RowChunk* __restrict__ tasks,
                                                           int counter) {
    ROWS_GATE(c);
    const int lane = threadIdx.x & 31;
    const int64_t nv4 = ((p.n + 31) / 32 + 3) / 4;
    const unsigned long long m = min(c.rc[counter], c.chunk_cap);
    uint4* out = c.elist + (MODE ? c.ecap : 0);
    for (unsigned long long t = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5; t < m;
         t += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
        const RowChunk tk = tasks[t];
        const DenseRule r = p.rules[tk.rule];
        const int X = MODE ? r.C : r.B;
        CFPQ_DASSERT(tk.row >= 0 && tk.row < p.n && tk.first >= 0);
        const uint4* row = reinterpret_cast<const uint4*>(p.T[X] + (size_t)tk.row * p.Wp);
        const unsigned long long base = (unsigned long long)(uint32_t)tk.first;
        const unsigned long long lim = base + (unsigned long long)tk.count;
        unsigned long long at0 = base;   // next slot (warp-uniform)
        for (int64_t v0 = 0; v0 < nv4; v0 += 32 * kCompactB) {
            uint4 x[kCompactB];
#pragma unroll
            for (int b = 0; b < kCompactB; ++b) {
                const int64_t v = v0 + (int64_t)b * 32 + lane;
                x[b] = v < nv4 ? __ldg(row + v) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < kCompactB; ++b) {
                const uint32_t wd[4] = {x[b].x, x[b].y, x[b].z, x[b].w};
                int cntl = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) cntl += MODE ? (wd[q] != 0u) : __popc(wd[q]);
                int incl = cntl;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (cntl) {
                    unsigned long long at = at0 + (unsigned long long)(incl - cntl);
                    const int64_t v = v0 + (int64_t)b * 32 + lane;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t bits = wd[q];
                        if (MODE) {
                            if (bits) {
                                if (at < lim && at < c.ecap)
                                    out[at] = make_uint4((uint32_t)tk.rule, (uint32_t)tk.row, (uint32_t)(4 * v + q), bits);
                                ++at;
                            }
                        } else {
                            while (bits) {
                                const int bt = __ffs(bits) - 1;
                                bits &= bits - 1u;
                                if (at < lim && at < c.ecap)
                                    out[at] = make_uint4((uint32_t)tk.rule, (uint32_t)tk.row,
                                                         (uint32_t)((4 * v + q) * 32 + bt), 1u);
                                ++at;
                            }
                        }
                    }
                }
                at0 += (unsigned long long)total;
            }
        }
        for (unsigned long long e = at0 + lane; e < lim; e += 32)
            if (e < c.ecap) out[e] = make_uint4(0, 0, 0, 0);
    }
}

// L entries {leader rule, i, r}: every rule A -> B C_g of the group, j in CSR_C_g(r).
__global__ void __launch_bounds__(256) rows_lmerge_kernel(DenseParams p, RowsCtx c, const int32_t* __restrict__ rule_out) {
    ROWS_GATE(c);
    const unsigned long long m = min(c.rc[5], c.ecap);
    unsigned long long my_new = 0;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < m;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const uint4 en = c.elist[e];
        if (!en.w) continue;
        const int i = (int)en.y, rr = (int)en.z;
        CFPQ_DASSERT(i < p.n && rr < p.n);
        for (int qq = (int)en.x; qq >= 0; qq = rows_l_follow(c.l_next[qq])) {
            // the ELL head {beg, deg, nb0, nb1} of CSR_C(r): one load for the usual <= 2 entries
            const int4 h = __ldg(c.nt[p.rules[qq].C].csr_ell + rr);
            const int A = rule_out[qq];
            for (int f2 = 0; f2 < h.y; ++f2) {
                const int j = f2 == 0 ? h.z : (f2 == 1 ? h.w : __ldg(c.adj_idx + h.x + f2));
                rows_merge(p, c, A, i, j >> 5, 1u << (j & 31), my_new);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if ((threadIdx.x & 31) == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// R entries {rule, r, word, bits}: OR bits into word `word` of every row i in CSC_B(r).
__global__ void __launch_bounds__(256) rows_rmerge_kernel(DenseParams p, RowsCtx c, const int32_t* __restrict__ rule_out) {
    ROWS_GATE(c);
    const unsigned long long m = min(c.rc[6], c.ecap);
    unsigned long long my_new = 0;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < m;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const uint4 en = c.elist[c.ecap + e];
        if (!en.w) continue;
        const int q = (int)en.x, rr = (int)en.y;
        CFPQ_DASSERT(rr < p.n && (int64_t)en.z < p.Wp);
        const int4 h = __ldg(c.nt[p.rules[q].B].csc_ell + rr);   // CSC_B(r): ELL head first
        const int A = rule_out[q];
        for (int f2 = 0; f2 < h.y; ++f2) {
            const int i = f2 == 0 ? h.z : (f2 == 1 ? h.w : __ldg(c.adj_idx + h.x + f2));
            rows_merge(p, c, A, i, (int64_t)en.z, en.w, my_new);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if ((threadIdx.x & 31) == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// Forms L and P: one warp per task of the plan's list: an L chunk (<= kChunkL set bits of one row of T_B)
// Latency-bound chains (CSR pointers -> index -> pre-check -> atomic): many warps resident.
__global__ void __launch_bounds__(256, 4) rows_scatter_kernel(DenseParams p, RowsCtx c, const int32_t* __restrict__ rule_out,
                                                              const RowChunk* __restrict__ tasks) {
    ROWS_GATE(c);
    __shared__ int32_t wlist[8][kChunkL];   // per warp: the chunk's selected set bits
    const int lane = threadIdx.x & 31;
    const int64_t wn = (p.n + 31) / 32;
    const unsigned long long m = min(c.rc[4], c.chunk_cap);
    unsigned long long my_new = 0;
    for (unsigned long long t = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5; t < m;
         t += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
        const RowChunk tk = tasks[t];
        const int i = tk.row, q = tk.rule;
        const DenseRule r = p.rules[q];
        const int A = rule_out[q];
        const int32_t* cptr = c.nt[r.C].csr_ptr;
        if (!c.nt[r.B].is_const) {
            // L: select the set bits of rank [first, first+count) of the bit row T_B[i]
            // (T_{k-1}; four 128-bit loads per lane in flight, warp prefix counts) into a
            // per-warp list, then every lane takes list entries: a hub row's bits spread over
            // many warps and all 32 lanes, not over the lanes that happen to hold its words
            const uint4* rowB = reinterpret_cast<const uint4*>(p.T[r.B] + (size_t)i * p.Wp);
            const int64_t nv4 = (wn + 3) / 4;
            int32_t* lst = wlist[threadIdx.x >> 5];
            int base = 0;   // set bits before the current batch
            for (int64_t v0 = lane; v0 - lane < nv4 && base < tk.first + tk.count; v0 += 32 * kScanBatch) {
                uint4 x[kScanBatch];
#pragma unroll
                for (int b = 0; b < kScanBatch; ++b)
                    x[b] = v0 + b * 32 < nv4 ? __ldg(rowB + v0 + b * 32) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int b = 0; b < kScanBatch; ++b) {
                    const int pc = __popc(x[b].x) + __popc(x[b].y) + __popc(x[b].z) + __popc(x[b].w);
                    int incl = pc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        int v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const int total = __shfl_sync(0xffffffffu, incl, 31);
                    int rank = base + incl - pc;
                    if (pc && rank < tk.first + tk.count && rank + pc > tk.first) {
                        const int64_t v = v0 + b * 32;
                        const uint32_t ws[4] = {x[b].x, x[b].y, x[b].z, x[b].w};
                        for (int h = 0; h < 4; ++h) {
                            uint32_t bits = ws[h];
                            while (bits) {
                                const int bit = __ffs(bits) - 1;
                                bits &= bits - 1u;
                                if (rank >= tk.first && rank < tk.first + tk.count) {
                                    CFPQ_DASSERT(rank - tk.first < kChunkL);
                                    lst[rank - tk.first] = (int)((v * 4 + h) * 32) + bit;
                                }
                                ++rank;
                            }
                        }
                    }
                    base += total;
                }
            }
            __syncwarp();
            // the plan sized the chunk from cnt[B][i], which a re-run of the shard (chunk-list
            // overflow) reads after this iteration's merges grew it: list only the bits found
            const int found = min(tk.count, max(0, base - tk.first));
            // every L rule of the group (same B, so the same listed bits): A -> B C_g
            for (int qq = q; qq >= 0; qq = rows_l_follow(c.l_next[qq])) {
                const int Ag = rule_out[qq];
                const int32_t* cp = c.nt[p.rules[qq].C].csr_ptr;
                for (int e = lane; e < found; e += 32) {
                    const int rr = lst[e];
                    const int e1 = __ldg(cp + rr + 1);
                    for (int f2 = __ldg(cp + rr); f2 < e1; ++f2) {
                        const int j = __ldg(c.adj_idx + f2);
                        rows_merge(p, c, Ag, i, j >> 5, 1u << (j & 31), my_new);
                    }
                }
            }
            __syncwarp();
        } else {
            // P: CSR_B(i) x CSR_C(r) (iteration 1 only)
            const int32_t* bptr = c.nt[r.B].csr_ptr;
            const int b1 = __ldg(bptr + i + 1);
            for (int e = __ldg(bptr + i) + lane; e < b1; e += 32) {
                const int rr = __ldg(c.adj_idx + e);
                const int e1 = __ldg(cptr + rr + 1);
                for (int f2 = __ldg(cptr + rr); f2 < e1; ++f2) {
                    const int j = __ldg(c.adj_idx + f2);
                    rows_merge(p, c, A, i, j >> 5, 1u << (j & 31), my_new);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// Forms R and V: one CTA per chunk ORs the chunk's bit rows T_C[r] (128-bit loads, 4 rows
// in flight per thread) into a register accumulator and merges its non-zero words.
template <int NV>   // uint4 accumulators per thread (>= ceil(row uint4s / kRowThreads))
__global__ void __launch_bounds__(kRowThreads) rows_gather_kernel(DenseParams p, RowsCtx c,
                                                                 const int32_t* __restrict__ rule_out,
                                                                 const RowChunk* __restrict__ chunks, int counter) {
    __shared__ int32_t list[kChunk];
    __shared__ int32_t wsum[kRowThreads / 32];
    __shared__ int32_t n_list;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wn = (p.n + 31) / 32;
    const int64_t nv4 = (wn + 3) / 4;
    const unsigned long long m = min(c.rc[counter], c.chunk_cap);
    unsigned long long my_new = 0;
    for (unsigned long long ci = blockIdx.x; ci < m; ci += gridDim.x) {
        const RowChunk ch = chunks[ci];
        const DenseRule r = p.rules[ch.rule];
        const uint32_t* TC = p.T[r.C];
        const uint32_t* cntC = c.cnt + (size_t)r.C * p.n;
        if (threadIdx.x == 0) n_list = 0;
        __syncthreads();
        if (!c.nt[r.B].is_const) {
            // V: the set bits of rank [first, first+count) of T_B[i], walked in 256-word slices
            const uint32_t* rowB = p.T[r.B] + (size_t)ch.row * p.Wp;
            int base = 0;
            for (int64_t w0 = 0; w0 < wn && base < ch.first + ch.count; w0 += kRowThreads) {
                int64_t w = w0 + threadIdx.x;
                uint32_t bits = w < wn ? __ldg(rowB + w) : 0u;
                int pc = __popc(bits);
                int incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                if (lane == 31) wsum[warp] = incl;
                __syncthreads();
                int before = 0, total = 0;
                for (int q = 0; q < kRowThreads / 32; ++q) {
                    if (q < warp) before += wsum[q];
                    total += wsum[q];
                }
                int rank = base + before + incl - pc;
                while (bits) {
                    int b = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    if (rank >= ch.first && rank < ch.first + ch.count) list[rank - ch.first] = (int32_t)(w * 32 + b);
                    ++rank;
                }
                base += total;
                __syncthreads();
            }
            // bits found (a re-run of the shard may have sized the chunk from a grown count)
            if (threadIdx.x == 0) n_list = min(ch.count, max(0, base - ch.first));
        } else {
            // R: CSR_B(i) entries [first, first+count), rows of T_C that are empty skipped
            if (threadIdx.x < ch.count) {
                const int rr = __ldg(c.adj_idx + __ldg(c.nt[r.B].csr_ptr + ch.row) + ch.first + threadIdx.x);
                if (cntC[rr]) list[atomicAdd(&n_list, 1)] = rr;
            }
        }
        __syncthreads();
        const int nl = n_list;
        uint4 acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = make_uint4(0, 0, 0, 0);
        int e = 0;
        for (; e + 4 <= nl; e += 4) {
            const uint4* r0 = reinterpret_cast<const uint4*>(TC + (size_t)list[e] * p.Wp);
            const uint4* r1 = reinterpret_cast<const uint4*>(TC + (size_t)list[e + 1] * p.Wp);
            const uint4* r2 = reinterpret_cast<const uint4*>(TC + (size_t)list[e + 2] * p.Wp);
            const uint4* r3 = reinterpret_cast<const uint4*>(TC + (size_t)list[e + 3] * p.Wp);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                int64_t g = (int64_t)v * kRowThreads + threadIdx.x;
                if (g < nv4) {
                    const uint4 x0 = __ldg(r0 + g), x1 = __ldg(r1 + g), x2 = __ldg(r2 + g), x3 = __ldg(r3 + g);
                    acc[v].x |= x0.x | x1.x | x2.x | x3.x;
                    acc[v].y |= x0.y | x1.y | x2.y | x3.y;
                    acc[v].z |= x0.z | x1.z | x2.z | x3.z;
                    acc[v].w |= x0.w | x1.w | x2.w | x3.w;
                }
            }
        }
        for (; e < nl; ++e) {
            const uint4* r0 = reinterpret_cast<const uint4*>(TC + (size_t)list[e] * p.Wp);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                int64_t g = (int64_t)v * kRowThreads + threadIdx.x;
                if (g < nv4) {
                    const uint4 x = __ldg(r0 + g);
                    acc[v].x |= x.x;
                    acc[v].y |= x.y;
                    acc[v].z |= x.z;
                    acc[v].w |= x.w;
                }
            }
        }
        const int A = rule_out[ch.rule];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            int64_t g = (int64_t)v * kRowThreads + threadIdx.x;
            if (g < nv4) {
                const uint32_t a[4] = {acc[v].x, acc[v].y, acc[v].z, acc[v].w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (a[q]) rows_merge(p, c, A, ch.row, 4 * g + q, a[q], my_new);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_new += __shfl_xor_sync(0xffffffffu, my_new, o);
    if (lane == 0 && my_new) atomicAdd(p.new_cells + p.n_nt, my_new);
}

// Row-block sharding of the bit-row engine (§8(e)).  Every rank keeps full replicas of
// T_{k-1} and T_k and derives only its rows [row_lo, row_hi); its Δ_k word list is exchanged
// and applied on every rank.  Applying a word ORs it into T_k and counts the bits it flips
// (into the new-cell total and the row popcounts): idempotent, so words a rank already holds
// (its own, or every shard's when the shards are emulated in one process) flip nothing.
__global__ void rows_apply_kernel(DenseParams p, RowsCtx c, unsigned long long begin, unsigned long long end) {
    unsigned long long flips = 0;
    for (unsigned long long e = begin + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < end;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const uint4 d = c.dlist[e];
        uint32_t* addr = p.Tn[d.x] + (size_t)d.y * p.Wp + d.z;
        if ((d.w & ~*addr) == 0) continue;
        const uint32_t fl = d.w & ~atomicOr(addr, d.w);
        if (fl) {
            atomicAdd(c.cnt + (size_t)d.x * p.n + d.y, (uint32_t)__popc(fl));
            flips += __popc(fl);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) flips += __shfl_xor_sync(0xffffffffu, flips, o);
    if ((threadIdx.x & 31) == 0 && flips) atomicAdd(p.new_cells + p.n_nt, flips);
}

// A shard's Δ_k word list after it overflowed: rebuild it from T_k minus T_{k-1} over the
// shard's rows (count = 1: only count the words that gained bits).  Runs only on overflow.
__global__ void rows_diff_kernel(DenseParams p, RowsCtx c, int count_only) {
    const int64_t wn = (p.n + 31) / 32;
    const int64_t per_nt = (int64_t)(c.row_hi - c.row_lo) * wn;
    const int64_t total = per_nt * p.n_out;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int o = (int)(t / per_nt);
        const int64_t rem = t - (int64_t)o * per_nt;
        const int i = c.row_lo + (int)(rem / wn);
        const int64_t w = rem - (int64_t)(i - c.row_lo) * wn;
        const int A = p.out_nt[o];
        const uint32_t d = p.Tn[A][(size_t)i * p.Wp + w] & ~p.T[A][(size_t)i * p.Wp + w];
        if (!d) continue;
        const unsigned long long at = atomicAdd(c.rc + 1, 1ull);
        if (!count_only && at < c.dlist_cap) c.dlist[at] = make_uint4((uint32_t)A, (uint32_t)i, (uint32_t)w, d);
    }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 2D uint8 tensor [rows][row_bytes] with a (128 x box_rows) box, 128B swizzle.
static bool make_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t row_bytes, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)kTK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

size_t dense_smem_bytes() { return (size_t)kStages * kStageBytes + 1024 + 256; }

struct DenseEngine {
    int32_t n = 0, np = 0, nt_tiles = 0, n_nt = 0;
    int64_t Wp = 0;
    bool fp4 = false;                              // kind::mxf4 e2m1 packs instead of int8
    std::vector<int32_t> is_const, packA, packB;   // packA[X]: X is a left operand (T8), packB: right (T8T)
    std::vector<int64_t> h_mapA, h_mapB;
    uint8_t* T8 = nullptr;
    uint8_t* T8T = nullptr;
    uint8_t* occ = nullptr;
    int64_t* mapA_row = nullptr;
    int64_t* mapB_row = nullptr;
    int32_t* out_nt = nullptr;
    int32_t* rule_ptr = nullptr;
    DenseRule* rules = nullptr;
    const uint32_t** Tptr = nullptr;
    uint32_t** Tnptr = nullptr;
    unsigned long long* new_cells = nullptr;
    int32_t n_out = 0;
    std::vector<int32_t> h_out;
    CUtensorMap tmA, tmB, tmBh;   // tmBh: 128-row box of T8T (CTA-pair halves)
    int grid = 0;
    unsigned long long kblocks_total = 0;
    uint32_t* cnt = nullptr;   // accounting scratch
    int32_t* rule_out = nullptr;               // [rules] output NT of each rule (bit-row path)
    int32_t* l_next = nullptr;                 // [rules] L-form groups by B (RowsCtx::l_next)
    std::vector<int32_t> h_rule_out;
    std::vector<int32_t> h_l_plan;
    void* chunks = nullptr;                    // bit-row path work list
    unsigned long long chunk_cap = 0;
    uint32_t* rcnt = nullptr;                  // bit-row path: per NT row popcounts
    std::vector<DenseRule> h_rules;            // rules in output order (host copy)
    bool forms_known = false, has_r = false, has_v = false;
    void* dlist = nullptr;                     // bit-row path: Δ_k word list (uint4)
    unsigned long long dlist_cap = 0;
    unsigned long long* rc = nullptr;          // bit-row path counters
    uint4* elist = nullptr;                    // bit-row compact mode: L / R entry lists [2 * ecap]
    unsigned long long ecap = 0;
    cudaStream_t side = nullptr;               // compact mode: the R pipeline runs beside the L one
    bool pipe = false;                         // pipelined iterations (rows_pipe_*)
    int* d_stop = nullptr;                     // pipelined iterations: device stop flag
    unsigned long long* h_map = nullptr;       // mapped pinned [2 slots][16]: outcome + counters
    unsigned long long* d_map = nullptr;       // its device alias
    bool pipe_enqueue = false;                 // inside rows_pipe_iteration
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int32_t launch_mode = 0;                   // cfpq_options.dense_launch
    int32_t rgather_variant = 0;               // diagnostics (diag_flags bits 4-6): R-form kernel shape
    unsigned long long* h_rc = nullptr;        // bit-row path counters, pinned host copy
    unsigned long long* h_new = nullptr;       // new-cell counters, pinned host copy (dense_finish)
    bool list_complete = true;                 // the Δ word list of the last iteration holds every word
    const NTInfo* rows_nt = nullptr;           // bit-row path: this iteration's NT table / CSR
    const int32_t* rows_adj = nullptr;
    bool rows_first = false;
    ~DenseEngine() {
        cudaFree(cnt);
        cudaFree(rule_out);
        cudaFree(l_next);
        if (h_rc) cudaFreeHost(h_rc);
        if (h_new) cudaFreeHost(h_new);
        cudaFree(chunks);
        cudaFree(rcnt);
        cudaFree(dlist);
        cudaFree(elist);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
        cudaFree(d_stop);
        if (h_map) cudaFreeHost(h_map);
        cudaFree(rc);
        cudaFree(T8); cudaFree(T8T); cudaFree(occ); cudaFree(mapA_row); cudaFree(mapB_row); cudaFree(out_nt);
        cudaFree(rule_ptr); cudaFree(rules); cudaFree(Tptr); cudaFree(Tnptr); cudaFree(new_cells);
    }
};

void dense_destroy(DenseEngine* e) { delete e; }
void dense_set_rgather_variant(DenseEngine* e, int v) { e->rgather_variant = v; }

DenseEngine* dense_create(int32_t n, int32_t n_nt, int64_t Wp, const std::vector<Rule3>& rules,
                          const std::vector<int32_t>& is_const, cudaStream_t s, std::string* err, bool tensor,
                          bool fp4, int64_t dlist_cap, int32_t launch_mode) {
    DenseEngine* e = new DenseEngine();
    e->fp4 = fp4;
    e->n = n;
    e->n_nt = n_nt;
    e->Wp = Wp;
    e->np = ((n + kTN - 1) / kTN) * kTN;
    if (e->np == 0) e->np = kTN;
    e->nt_tiles = e->np / kTM;
    e->is_const = is_const;
    e->packA.assign(n_nt, 0);
    e->packB.assign(n_nt, 0);
    std::vector<std::vector<DenseRule>> by(n_nt);
    for (auto& r : rules) {
        by[r.A].push_back(DenseRule{r.A, r.B, r.C, 0});
        e->packA[r.B] = 1;
        e->packB[r.C] = 1;
    }
    std::vector<int32_t> rp(1, 0);
    std::vector<DenseRule> rl;
    for (int A = 0; A < n_nt; ++A) {
        if (by[A].empty()) continue;
        e->h_out.push_back(A);
        for (auto& r : by[A]) rl.push_back(r);
        rp.push_back((int32_t)rl.size());
    }
    e->n_out = (int32_t)e->h_out.size();
    if (!tensor) {
        std::fill(e->packA.begin(), e->packA.end(), 0);
        std::fill(e->packB.begin(), e->packB.end(), 0);
    }
    int na = 0, nb = 0;
    e->h_mapA.assign(n_nt, -1);
    e->h_mapB.assign(n_nt, -1);
    for (int X = 0; X < n_nt; ++X) {
        if (e->packA[X]) e->h_mapA[X] = (int64_t)(na++) * e->np;
        if (e->packB[X]) e->h_mapB[X] = (int64_t)(nb++) * e->np;
    }
    auto fail = [&](const char* what, cudaError_t c) {
        if (err) *err = std::string("dense engine: ") + what + ": " + cudaGetErrorString(c);
        cudaGetLastError();
        delete e;
        return (DenseEngine*)nullptr;
    };
    const size_t pack = (size_t)e->np * e->np;
    cudaError_t c;
    if ((c = cudaMalloc(&e->T8, std::max<size_t>(1, pack * na))) != cudaSuccess) return fail("T8", c);
    if ((c = cudaMalloc(&e->T8T, std::max<size_t>(1, pack * nb))) != cudaSuccess) return fail("T8T", c);
    if ((c = cudaMalloc(&e->occ, (size_t)n_nt * e->nt_tiles * e->nt_tiles)) != cudaSuccess) return fail("occ", c);
    if ((c = cudaMemsetAsync(e->occ, 0, (size_t)n_nt * e->nt_tiles * e->nt_tiles, s)) != cudaSuccess) return fail("occ", c);
    if ((c = cudaMalloc(&e->mapA_row, n_nt * 8)) != cudaSuccess) return fail("maps", c);
    if ((c = cudaMalloc(&e->mapB_row, n_nt * 8)) != cudaSuccess) return fail("maps", c);
    if ((c = cudaMalloc(&e->out_nt, std::max(1, e->n_out) * 4)) != cudaSuccess) return fail("tables", c);
    if ((c = cudaMalloc(&e->rule_ptr, rp.size() * 4)) != cudaSuccess) return fail("tables", c);
    if ((c = cudaMalloc(&e->rules, std::max<size_t>(1, rl.size()) * sizeof(DenseRule))) != cudaSuccess) return fail("tables", c);
    if ((c = cudaMalloc(&e->Tptr, n_nt * sizeof(void*))) != cudaSuccess) return fail("tables", c);
    if ((c = cudaMalloc(&e->Tnptr, n_nt * sizeof(void*))) != cudaSuccess) return fail("tables", c);
    if ((c = cudaMalloc(&e->new_cells, (n_nt + 2) * 8)) != cudaSuccess) return fail("counters", c);
    cudaMemcpyAsync(e->mapA_row, e->h_mapA.data(), n_nt * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(e->mapB_row, e->h_mapB.data(), n_nt * 8, cudaMemcpyHostToDevice, s);
    if (e->n_out) cudaMemcpyAsync(e->out_nt, e->h_out.data(), e->n_out * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(e->rule_ptr, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, s);
    if (!rl.empty()) cudaMemcpyAsync(e->rules, rl.data(), rl.size() * sizeof(DenseRule), cudaMemcpyHostToDevice, s);
    for (auto& r : rl) e->h_rule_out.push_back(r.A);
    e->h_rules = rl;
    if ((c = cudaMalloc(&e->rule_out, std::max<size_t>(1, rl.size()) * 4)) != cudaSuccess) return fail("tables", c);
    if (!rl.empty())
        cudaMemcpyAsync(e->rule_out, e->h_rule_out.data(), rl.size() * 4, cudaMemcpyHostToDevice, s);
    {
        // L-form rules (B changes, C preterminal) grouped by B, in rule order: the leader owns
        // the row scan and links to the next member (>= 0, or -1 if alone); member q links
        // to the next one as -(next + 3), or -2 if last (RowsCtx::l_next, rows_l_follow)
        std::vector<std::vector<int32_t>> groups(n_nt);
        for (size_t q = 0; q < rl.size(); ++q)
            if (!is_const[rl[q].B] && is_const[rl[q].C]) groups[rl[q].B].push_back((int32_t)q);
        e->h_l_plan.assign(rl.size(), -1);
        for (auto& gq : groups)
            for (size_t t = 0; t < gq.size(); ++t) {
                const bool has_next = t + 1 < gq.size();
                if (t == 0) e->h_l_plan[gq[t]] = has_next ? gq[t + 1] : -1;
                else e->h_l_plan[gq[t]] = has_next ? -(gq[t + 1] + 3) : -2;
            }
    }
    if ((c = cudaMalloc(&e->l_next, std::max<size_t>(1, rl.size()) * 4)) != cudaSuccess) return fail("tables", c);
    if (!rl.empty())
        cudaMemcpyAsync(e->l_next, e->h_l_plan.data(), rl.size() * 4, cudaMemcpyHostToDevice, s);
    const int64_t row_bytes = fp4 ? e->np / 2 : e->np;   // nibble packs: half the bytes per row
    if (!make_map(&e->tmA, e->T8, (int64_t)std::max(na, 1) * e->np, row_bytes, kTM) ||
        !make_map(&e->tmB, e->T8T, (int64_t)std::max(nb, 1) * e->np, row_bytes, kTN) ||
        !make_map(&e->tmBh, e->T8T, (int64_t)std::max(nb, 1) * e->np, row_bytes, kTN / 2)) {
        if (err) *err = "dense engine: cuTensorMapEncodeTiled failed";
        delete e;
        return nullptr;
    }
    if ((c = cudaFuncSetAttribute(dense_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_smem_bytes())) != cudaSuccess) {
        if (err) *err = std::string("dense kernel smem attribute: ") + cudaGetErrorString(c);
        delete e;
        return nullptr;
    }
    if ((c = cudaFuncSetAttribute(dense_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dense_smem_bytes())) !=
        cudaSuccess)
        return fail("smem attribute", c);
    if ((c = cudaFuncSetAttribute(dense_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_smem_bytes())) != cudaSuccess)
        return fail("smem attribute", c);
    if ((c = cudaFuncSetAttribute(dense_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_smem_bytes())) != cudaSuccess)
        return fail("smem attribute", c);
    if ((c = cudaFuncSetAttribute(dense2sm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense2_smem_bytes())) != cudaSuccess)
        return fail("smem attribute", c);
    if ((c = cudaFuncSetAttribute(dense2sm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense2_smem_bytes())) != cudaSuccess)
        return fail("smem attribute", c);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int total = e->n_out * (e->np / kTM) * (e->np / kTN);
    e->grid = std::max(1, std::min(sms, total));
    e->launch_mode = launch_mode;
    e->dlist_cap = dlist_cap > 0 ? (unsigned long long)dlist_cap : (1ull << 20);   // bit-row Δ_k word list
    // compact-mode entry lists start at 2^21 entries each, or at the caller's (small) list
    // capacity, so that the tests exercise their overflow-and-redo path
    e->ecap = dlist_cap > 0 && dlist_cap < (1 << 21) ? std::max<unsigned long long>(64, dlist_cap) : (1ull << 21);
    return e;
}

// One Jacobi iteration in three parts (so that a multi-GPU exchange can sit between the
// product and the read-back): begin = packs of the operands of T_{k-1} + counter reset;
// product = T_k rows of row tiles [i_lo, i_hi) of every output; finish = read the new-cell
// counters (device -> host).
cudaError_t dense_begin(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, bool first, cudaStream_t s,
                        int* launches, bool pack_operands) {
    const size_t pack = (size_t)e->np * e->np / (e->fp4 ? 2 : 1);   // bytes per packed NT
    for (int X = 0; X < e->n_nt && pack_operands; ++X) {
        if (!(e->packA[X] || e->packB[X])) continue;
        if (!first && e->is_const[X]) continue;   // preterminals never change after seeding
        uint8_t* a = e->packA[X] ? e->T8 + (size_t)(e->h_mapA[X] / e->np) * pack : nullptr;
        uint8_t* b = e->packB[X] ? e->T8T + (size_t)(e->h_mapB[X] / e->np) * pack : nullptr;
        dim3 grid(e->nt_tiles, e->nt_tiles);
        uint8_t* oc = e->occ + (size_t)X * e->nt_tiles * e->nt_tiles;
        if (e->fp4) pack_kernel<true><<<grid, 128, 0, s>>>(T[X], e->n, e->Wp, e->np, a, b, oc, e->nt_tiles);
        else pack_kernel<false><<<grid, 128, 0, s>>>(T[X], e->n, e->Wp, e->np, a, b, oc, e->nt_tiles);
        if (launches) ++*launches;
    }
    cudaError_t c;
    if ((c = cudaGetLastError()) != cudaSuccess) return c;
    if ((c = cudaMemcpyAsync((void*)e->Tptr, T, e->n_nt * sizeof(void*), cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return c;
    if ((c = cudaMemcpyAsync((void*)e->Tnptr, Tn, e->n_nt * sizeof(void*), cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return c;
    return cudaMemsetAsync(e->new_cells, 0, (e->n_nt + 2) * 8, s);
}

cudaError_t dense_product(DenseEngine* e, int64_t i_lo, int64_t i_hi, cudaStream_t s, int* launches, int64_t j_lo,
                          int64_t j_hi) {
    if (j_hi < 0) j_hi = e->np / kTN;
    if (e->n_out == 0 || i_hi <= i_lo || j_hi <= j_lo) return cudaSuccess;
    DenseParams p{};
    p.n = e->n;
    p.np = e->np;
    p.Wp = e->Wp;
    p.n_out = e->n_out;
    p.out_nt = e->out_nt;
    p.rule_ptr = e->rule_ptr;
    p.rules = e->rules;
    p.T = e->Tptr;
    p.Tn = e->Tnptr;
    p.occ = e->occ;
    p.nt_tiles = e->nt_tiles;
    p.new_cells = e->new_cells;
    p.n_nt = e->n_nt;
    p.i_lo = (int32_t)i_lo;
    p.i_hi = (int32_t)i_hi;
    p.j_lo = (int32_t)j_lo;
    p.j_hi = (int32_t)j_hi;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // cfpq_options.dense_launch: CTA pairs with one M = 256 UMMA per pair (cta_group::2) by
    // default (config S, n = 16,384: fp4 10.3 vs 10.7 ms one CTA per SM, int8 18.0 vs 20.5
    // ms); CTA pairs sharing a multicast B tile measured 18% SLOWER than one CTA per SM (31.6
    // vs 26.7 ms: the pair runs in lockstep and a 2-CTA multicast saves no L2 traffic, cf.
    // B300_MICROARCH "TMA-MC at csz <= 4, MC ~ UC")
    const bool pair = e->launch_mode == 3;
    const bool two_sm = e->launch_mode == 0 || e->launch_mode == 1;
    const bool use2 = two_sm && sms >= 2 && !pair;
    if (use2) {
        const int64_t units = (int64_t)e->n_out * ((i_hi - i_lo + 1) / 2) * (j_hi - j_lo);
        const int grid = (int)std::max<int64_t>(2, std::min<int64_t>(sms / 2, units) * 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kDenseThreads);
        cfg.dynamicSmemBytes = dense2_smem_bytes();
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t c = e->fp4 ? cudaLaunchKernelEx(&cfg, dense2sm_kernel<true>, p, e->tmA, e->tmBh,
                                                    (const int64_t*)e->mapA_row, (const int64_t*)e->mapB_row)
                               : cudaLaunchKernelEx(&cfg, dense2sm_kernel<false>, p, e->tmA, e->tmBh,
                                                    (const int64_t*)e->mapA_row, (const int64_t*)e->mapB_row);
        if (launches) ++*launches;
        return c != cudaSuccess ? c : cudaGetLastError();
    }
    if (pair && sms >= 2) {
        // CTA pairs (clusters of 2) share the B tile through TMA multicast
        const int64_t units = (int64_t)e->n_out * ((i_hi - i_lo + 1) / 2) * (j_hi - j_lo);
        const int grid = (int)std::max<int64_t>(2, std::min<int64_t>(sms / 2, units) * 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kDenseThreads);
        cfg.dynamicSmemBytes = dense_smem_bytes();
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t c = e->fp4 ? cudaLaunchKernelEx(&cfg, dense_kernel<2, true>, p, e->tmA, e->tmBh,
                                                    (const int64_t*)e->mapA_row, (const int64_t*)e->mapB_row)
                               : cudaLaunchKernelEx(&cfg, dense_kernel<2>, p, e->tmA, e->tmBh, (const int64_t*)e->mapA_row,
                                                    (const int64_t*)e->mapB_row);
        if (launches) ++*launches;
        return c != cudaSuccess ? c : cudaGetLastError();
    }
    const int64_t total = (int64_t)e->n_out * (i_hi - i_lo) * (j_hi - j_lo);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, total));
    if (e->fp4)
        dense_kernel<1, true><<<grid, kDenseThreads, dense_smem_bytes(), s>>>(p, e->tmA, e->tmB, e->mapA_row, e->mapB_row);
    else
        dense_kernel<1><<<grid, kDenseThreads, dense_smem_bytes(), s>>>(p, e->tmA, e->tmB, e->mapA_row, e->mapB_row);
    if (launches) ++*launches;
    return cudaGetLastError();
}

// grid = resident CTAs (grid-stride kernels: no queue of CTAs that start late)
template <typename K>
static int resident_grid(K kernel, int threads, int sms) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0) != cudaSuccess || per < 1) per = 1;
    return sms * per;
}

// 2-D block exchange staging (rows [r_lo, r_hi) x words [w_lo, w_hi) <-> contiguous buffer).
__global__ void bit_block_copy_kernel(uint32_t* T, int64_t Wp, int64_t r_lo, int64_t rows, int64_t w_lo, int64_t words,
                                      uint32_t* buf, int to_buf) {
    const int64_t total = rows * words;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / words, w = t - r * words;
        uint32_t* m = T + (size_t)(r_lo + r) * Wp + w_lo + w;
        if (to_buf) buf[t] = *m;
        else *m = buf[t];
    }
}

cudaError_t bit_block_copy(uint32_t* T, int64_t Wp, int64_t r_lo, int64_t r_hi, int64_t w_lo, int64_t w_hi,
                           uint32_t* buf, int to_buf, cudaStream_t s) {
    if (r_hi <= r_lo || w_hi <= w_lo) return cudaSuccess;
    const int64_t total = (r_hi - r_lo) * (w_hi - w_lo);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    bit_block_copy_kernel<<<grid, 256, 0, s>>>(T, Wp, r_lo, r_hi - r_lo, w_lo, w_hi - w_lo, buf, to_buf);
    return cudaGetLastError();
}

static DenseParams rows_params(DenseEngine* e) {
    DenseParams p{};
    p.n = e->n;
    p.np = e->np;
    p.Wp = e->Wp;
    p.n_out = e->n_out;
    p.out_nt = e->out_nt;
    p.rule_ptr = e->rule_ptr;
    p.rules = e->rules;
    p.T = e->Tptr;
    p.Tn = e->Tnptr;
    p.new_cells = e->new_cells;
    p.n_nt = e->n_nt;
    return p;
}

static int device_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Start of a bit-row iteration: T_k buffer := T_{k-1} (seed cells at iteration 1, else
// T_{k-2} | Δ_{k-1} words), Δ_k list and chunk counters reset.
cudaError_t rows_begin(DenseEngine* e, const NTInfo* nt, const int32_t* adj_idx, const uint64_t* log,
                       unsigned long long n_seeds, bool first, cudaStream_t s, int* launches) {
    if (e->n_out == 0) return cudaSuccess;
    if ((e->n + 31) / 32 > (int64_t)kRowMaxV4 * 4 * kRowThreads) return cudaErrorInvalidValue;
    cudaError_t c;
    const int32_t n_rules = (int32_t)e->h_rule_out.size();
    if (!e->rcnt) {
        if ((c = cudaMalloc(&e->rcnt, (size_t)e->n_nt * std::max(e->n, 1) * 4)) != cudaSuccess) return c;
        if ((c = cudaMalloc(&e->rc, 8 * 8)) != cudaSuccess) return c;
        if ((c = cudaMemsetAsync(e->rc, 0, 8 * 8, s)) != cudaSuccess) return c;
        if ((c = cudaMalloc(&e->dlist, e->dlist_cap * sizeof(uint4))) != cudaSuccess) return c;
        if ((c = cudaMallocHost(&e->h_rc, 8 * 8)) != cudaSuccess) return c;
        memset(e->h_rc, 0, 8 * 8);
    }
    // chunk capacity: grow lazily (the plan reports the exact count)
    const unsigned long long want = std::max<unsigned long long>(e->chunk_cap, (unsigned long long)n_rules * e->n + 1024);
    if (want > e->chunk_cap) {
        cudaFree(e->chunks);
        if ((c = cudaMalloc(&e->chunks, 3 * want * sizeof(RowChunk))) != cudaSuccess) return c;   // lists R, V, L/P
        e->chunk_cap = want;
    }
    if (!e->forms_known) {
        for (size_t q = 0; q < e->h_rules.size(); ++q) {
            const bool bc = e->is_const[e->h_rules[q].B], cc = e->is_const[e->h_rules[q].C];
            e->has_r |= bc && !cc;
            e->has_v |= !bc && !cc;
        }
        e->forms_known = true;
    }
    e->rows_nt = nt;
    e->rows_adj = adj_idx;
    e->rows_first = first;
    DenseParams p = rows_params(e);
    RowsCtx rc{nt, adj_idx, e->rcnt, (uint4*)e->dlist, e->dlist_cap, e->rc, first ? 1 : 0, n_rules, 0, e->n, e->l_next,
               e->chunk_cap, 0, 0, nullptr, 0, e->pipe ? e->d_stop : nullptr};
    const int sms = device_sms();
    // T_k buffer := T_{k-1}
    if (first) {
        if ((c = cudaMemsetAsync(e->rcnt, 0, (size_t)e->n_nt * e->n * 4, s)) != cudaSuccess) return c;
        if ((c = cudaMemsetAsync(e->rc, 0, 8 * 8, s)) != cudaSuccess) return c;
        if (n_seeds) rows_seed_kernel<<<sms * 8, 256, 0, s>>>(p, rc, log, n_seeds);
        e->list_complete = true;
    } else {
        rows_delta_kernel<<<sms * 8, 256, 0, s>>>(p, rc, e->list_complete ? 0 : 1);
        e->list_complete = true;
    }
    if (launches) *launches += 1;
    // Δ_k list and chunk counters restart
    rows_reset_kernel<<<1, 32, 0, s>>>(e->rc, 1, e->pipe ? e->d_stop : nullptr);
    return cudaGetLastError();
}

// Plan + products of the rows [row_lo, row_hi) of every output (all rows: one GPU).  Δ_k
// words are appended to the list after the ones already there (earlier emulated shards).
cudaError_t rows_shard(DenseEngine* e, int64_t row_lo, int64_t row_hi, cudaStream_t s, int* launches) {
    if (e->n_out == 0 || row_hi <= row_lo) return cudaSuccess;
    cudaError_t c;
    const int32_t n_rules = (int32_t)e->h_rule_out.size();
    DenseParams p = rows_params(e);
    // form R pushes input rows (each non-empty T_C row streamed once) on unsharded runs; row
    // shards gather their own output rows (rgather variants 1-4 and 7 force the gather, A/B)
    const bool push = row_lo == 0 && row_hi == e->n && (e->rgather_variant == 0 || e->rgather_variant == 5 ||
                                                         e->rgather_variant == 6);
    // compact mode (default on unsharded runs without rules whose two operands change): whole
    // operand rows streamed into entry lists, entries merged by one thread each (variant 0)
    const bool compact = push && !e->has_v && e->rgather_variant == 0;
    if (compact && !e->elist) {
        if ((c = cudaMalloc(&e->elist, 2 * e->ecap * sizeof(uint4))) != cudaSuccess) return c;
    }
    if (compact && !e->side) {
        if ((c = cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking)) != cudaSuccess) return c;
        if ((c = cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming)) != cudaSuccess) return c;
        if ((c = cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming)) != cudaSuccess) return c;
    }
    RowsCtx rc{e->rows_nt, e->rows_adj, e->rcnt, (uint4*)e->dlist, e->dlist_cap, e->rc, e->rows_first ? 1 : 0,
               n_rules, (int32_t)row_lo, (int32_t)row_hi, e->l_next, e->chunk_cap, push ? 1 : 0,
               compact ? 1 : 0, e->elist, compact ? e->ecap : 0, e->pipe ? e->d_stop : nullptr};
    const int sms = device_sms();
    // plan and products back to back, no host round trip: the products clamp every list to
    // its capacity and the counters are copied to pinned host memory behind them; the host
    // checks them after the iteration's synchronisation (rows_shard_check) and re-runs the
    // shard if a list overflowed (products are idempotent ORs; Δ_k records only new flips)
    if (!e->pipe_enqueue)   // (a pipelined iteration's rows_begin has just reset them)
        rows_reset_kernel<<<1, 32, 0, s>>>(e->rc, 0, e->pipe ? e->d_stop : nullptr);   // chunk lists, entry slots
    rows_plan_kernel<<<sms * 8, 256, 0, s>>>(p, rc, (RowChunk*)e->chunks, e->chunk_cap);
    // 4 CTAs x 8 warps per SM (measured: 6 or 8 CTAs with fewer registers are not faster)
    if (!compact)   // (compact mode lists P rules with the L rows)
    rows_scatter_kernel<<<resident_grid(rows_scatter_kernel, 256, sms), 256, 0, s>>>(p, rc, e->rule_out,
                                                                                 (const RowChunk*)e->chunks + 2 * e->chunk_cap);
    const int64_t nv4 = ((e->n + 31) / 32 + 3) / 4;
    const int nv = (int)((nv4 + kRowThreads - 1) / kRowThreads);
    const RowChunk* chR = (const RowChunk*)e->chunks;
    const RowChunk* chV = chR + e->chunk_cap;
    auto cta_gather = [&](const RowChunk* ch, int counter) {
        if (nv <= 1) rows_gather_kernel<1><<<sms * 8, kRowThreads, 0, s>>>(p, rc, e->rule_out, ch, counter);
        else if (nv <= 2) rows_gather_kernel<2><<<sms * 8, kRowThreads, 0, s>>>(p, rc, e->rule_out, ch, counter);
        else if (nv <= 4) rows_gather_kernel<4><<<sms * 8, kRowThreads, 0, s>>>(p, rc, e->rule_out, ch, counter);
        else rows_gather_kernel<8><<<sms * 8, kRowThreads, 0, s>>>(p, rc, e->rule_out, ch, counter);
    };
    if (compact) {
        // L: tasks in the V slot (rc[3]) -> entries [0, rc[5]); R: tasks in the R slot (rc[0]) ->
        // entries [ecap, ecap + rc[6]); then the merges.  The R pipeline runs on a side stream
        // beside the L one: each is a bandwidth-bound stream followed by latency-bound merges,
        // and the two overlap (they read T_{k-1} and OR into T_k with idempotent atomics)
        if (e->has_r) {
            if ((c = cudaEventRecord(e->ev_fork, s)) != cudaSuccess) return c;
            if ((c = cudaStreamWaitEvent(e->side, e->ev_fork, 0)) != cudaSuccess) return c;
            rows_compact_kernel<1><<<sms * 8, 256, 0, e->side>>>(p, rc, chR, 0);
            rows_rmerge_kernel<<<sms * 16, 256, 0, e->side>>>(p, rc, e->rule_out);
            if ((c = cudaEventRecord(e->ev_join, e->side)) != cudaSuccess) return c;
        }
        rows_compact_kernel<0><<<sms * 8, 256, 0, s>>>(p, rc, chV, 3);
        rows_lmerge_kernel<<<sms * 16, 256, 0, s>>>(p, rc, e->rule_out);
        if (e->has_r && (c = cudaStreamWaitEvent(s, e->ev_join, 0)) != cudaSuccess) return c;
        if (launches) *launches += e->has_r ? 4 : 2;
    }
    if (e->has_v && !compact) cta_gather(chV, 3);
    if (e->has_r && !compact) {
        // R chunks: a warp per (chunk, row slice of 32 x NVW uint4): many light warps
        // (config 4, one row in flight: 2 uint4 per lane 10.2 ms closure; 4 / 8 / 16: 10.7 /
        // 11.8 / 16.0 ms; 1: 11.5 ms); variants with RU rows in flight (rgather_variant)
        auto rg = [&](auto kern) {
            kern<<<resident_grid(kern, 256, sms), 256, 0, s>>>(p, rc, e->rule_out, chR);
        };
        // default: 2 uint4 per lane, 2 rows in flight, 6 CTAs/SM (config 4: 9.03-9.08 ms loop in
        // four runs vs 9.27-9.28 with one row in flight; 4 or 8 rows in flight lose occupancy)
        if (push) {
            switch (e->rgather_variant) {
                case 5: rg(rows_rpush_kernel<1, 8>); break;
                case 6: rg(rows_rpush_kernel<4, 4>); break;
                default: rg(rows_rpush_kernel<2, 6>); break;
            }
        } else {
            switch (e->rgather_variant) {
                case 1: rg(rows_rgather_kernel<1, 4, 6>); break;
                case 2: rg(rows_rgather_kernel<2, 1, 8>); break;
                case 3: rg(rows_rgather_kernel<2, 4, 4>); break;
                case 4: rg(rows_rgather_kernel<1, 8, 4>); break;
                default: rg(rows_rgather_kernel<2, 2, 6>); break;
            }
        }
    }
    if (launches) *launches += 2 + (e->has_v ? 1 : 0) + (e->has_r ? 1 : 0);
    // (pipelined iterations: rows_end_kernel writes the counters into mapped host memory)
    if (!e->pipe_enqueue && (c = cudaMemcpyAsync(e->h_rc, e->rc, 7 * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return c;
    return cudaGetLastError();
}

// After the stream passed rows_shard: grow what overflowed.  *redo = a chunk list did not
// fit (the shard must run again for the same rows); a Δ_k word list overflow of the previous
// iteration (the delta kernel copied whole matrices instead) only grows the list.
cudaError_t rows_shard_check(DenseEngine* e, cudaStream_t s, bool* redo, bool check_list) {
    cudaError_t c;
    (void)s;
    *redo = false;
    if (e->n_out == 0 || !e->rc) return cudaSuccess;
    const unsigned long long* got = e->h_rc;
    if (check_list && got[1] > e->dlist_cap) {
        // the Δ_k word list overflowed (words lost): the next iteration builds T_{k+1}'s buffer
        // by a whole-matrix copy, and the list grows for the iterations after
        cudaFree(e->dlist);
        e->dlist = nullptr;
        e->dlist_cap = std::max<unsigned long long>(e->dlist_cap * 4, got[1] + got[1] / 4);
        if ((c = cudaMalloc(&e->dlist, e->dlist_cap * sizeof(uint4))) != cudaSuccess) return c;
        e->list_complete = false;
    }
    const unsigned long long need = std::max(got[0], std::max(got[3], got[4]));
    if (need > e->chunk_cap) {
        cudaFree(e->chunks);
        e->chunk_cap = need + need / 4;
        if ((c = cudaMalloc(&e->chunks, 3 * e->chunk_cap * sizeof(RowChunk))) != cudaSuccess) return c;
        *redo = true;
    }
    // compact mode: an entry list that ran out (slots are task offsets: keep them < 2^31)
    const unsigned long long eneed = std::max(got[5], got[6]);
    if (e->elist && eneed > e->ecap) {
        if (eneed >= (1ull << 31)) return cudaErrorInvalidValue;
        cudaFree(e->elist);
        e->elist = nullptr;
        e->ecap = std::min<unsigned long long>(eneed + eneed / 4, (1ull << 31) - 1);
        if ((c = cudaMalloc(&e->elist, 2 * e->ecap * sizeof(uint4))) != cudaSuccess) return c;
        *redo = true;
    }
    return cudaSuccess;
}

cudaError_t rows_product(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, const NTInfo* nt,
                         const int32_t* adj_idx, const uint64_t* log, unsigned long long n_seeds, bool first,
                         cudaStream_t s, int* launches) {
    (void)T;
    (void)Tn;   // the kernels read the device copies set by dense_begin
    cudaError_t c = rows_begin(e, nt, adj_idx, log, n_seeds, first, s, launches);
    if (c != cudaSuccess) return c;
    return rows_shard(e, 0, e->n, s, launches);
}

// Sharded runs: the list length after a shard's products (host read, synchronises); when
// the list overflowed, the shard's words are rebuilt from T_k minus T_{k-1} into a grown list
// (the entries [0, keep) of earlier emulated shards are kept).
cudaError_t rows_list_settle(DenseEngine* e, int64_t row_lo, int64_t row_hi, unsigned long long keep, cudaStream_t s,
                             unsigned long long* count) {
    cudaError_t c;
    unsigned long long m = 0;
    *count = keep;
    if (e->n_out == 0 || !e->rc) return cudaSuccess;   // no binary rule: nothing derived
    if ((c = cudaMemcpyAsync(&m, e->rc + 1, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return c;
    if ((c = cudaStreamSynchronize(s)) != cudaSuccess) return c;
    if (m > e->dlist_cap) {
        const unsigned long long cap = std::max<unsigned long long>(e->dlist_cap * 2, m + m / 4 + 1024);
        void* nl = nullptr;
        if ((c = cudaMalloc(&nl, cap * sizeof(uint4))) != cudaSuccess) return c;
        if (keep && (c = cudaMemcpyAsync(nl, e->dlist, keep * sizeof(uint4), cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
            return c;
        if ((c = cudaStreamSynchronize(s)) != cudaSuccess) return c;
        cudaFree(e->dlist);
        e->dlist = nl;
        e->dlist_cap = cap;
        if ((c = cudaMemcpyAsync(e->rc + 1, &keep, 8, cudaMemcpyHostToDevice, s)) != cudaSuccess) return c;
        DenseParams p = rows_params(e);
        RowsCtx rc{e->rows_nt, e->rows_adj, e->rcnt, (uint4*)e->dlist, e->dlist_cap, e->rc, 0,
                   (int32_t)e->h_rule_out.size(), (int32_t)row_lo, (int32_t)row_hi, e->l_next, e->chunk_cap};
        rows_diff_kernel<<<device_sms() * 8, 256, 0, s>>>(p, rc, 0);
        if ((c = cudaMemcpyAsync(&m, e->rc + 1, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return c;
        if ((c = cudaStreamSynchronize(s)) != cudaSuccess) return c;
        if (m > e->dlist_cap) return cudaErrorMemoryAllocation;
    }
    *count = m;
    return cudaGetLastError();
}

// The Δ_k word list (uint4 {A, i, word, bits}) for the exchange; `ensure` grows it (content
// not kept) to hold `want` words.
cudaError_t rows_list(DenseEngine* e, unsigned long long want, void** list, unsigned long long* cap) {
    if (want > e->dlist_cap || !e->dlist) {
        cudaFree(e->dlist);
        e->dlist = nullptr;
        const unsigned long long nc = want + want / 4 + 1024;
        cudaError_t c = cudaMalloc(&e->dlist, nc * sizeof(uint4));
        if (c != cudaSuccess) return c;
        e->dlist_cap = nc;
    }
    *list = e->dlist;
    *cap = e->dlist_cap;
    return cudaSuccess;
}

// After the exchange: the list holds every rank's words [0, total); apply them to T_k.
cudaError_t rows_apply_all(DenseEngine* e, unsigned long long total, cudaStream_t s, int* launches) {
    cudaError_t c;
    if (e->n_out == 0 || !e->rc) return cudaSuccess;
    if ((c = cudaMemcpyAsync(e->rc + 1, &total, 8, cudaMemcpyHostToDevice, s)) != cudaSuccess) return c;
    if (total == 0) return cudaSuccess;
    DenseParams p = rows_params(e);
    RowsCtx rc{e->rows_nt, e->rows_adj, e->rcnt, (uint4*)e->dlist, e->dlist_cap, e->rc, 0,
               (int32_t)e->h_rule_out.size(), 0, e->n, e->l_next, e->chunk_cap};
    rows_apply_kernel<<<device_sms() * 8, 256, 0, s>>>(p, rc, 0ull, total);
    if (launches) *launches += 1;
    return cudaGetLastError();
}

// ---- pipelined bit-row iterations (unsharded compact mode) ----
// Iteration k+1 is enqueued before the host reads iteration k's outcome, so the host round
// trip of iteration k overlaps the products of k+1.  rows_end_kernel closes each iteration on
// the device: it records the new-cell count, and sets the stop flag at the fixpoint (no new
// cell), at the iteration cap, or when a chunk / entry list ran out (the host then redoes
// that iteration with grown lists, exactly as the unpipelined loop does); the speculative next
// iteration then does nothing.
__global__ void rows_end_kernel(RowsCtx c, unsigned long long* new_cells, int n_nt, unsigned long long chunk_cap,
                                unsigned long long ecap, int* stop, unsigned long long* out, long long k,
                                long long cap_iter, const uint32_t** Tptr, uint32_t** Tnptr, const int32_t* out_nt,
                                int n_out) {
    if (threadIdx.x != 0) return;
    if (*(volatile int*)stop) {
        out[0] = ~0ull;   // this iteration did not run
        out[1] = (unsigned long long)*(volatile int*)stop;
        return;
    }
    const unsigned long long nw = new_cells[n_nt];
    out[0] = nw;
    out[2] = c.rc[1];   // Δ_k words (the host grows the list when it ran out)
    for (int q = 0; q < 7; ++q) out[4 + q] = c.rc[q];
    int st = 0;
    if (c.rc[0] > chunk_cap || c.rc[3] > chunk_cap || c.rc[4] > chunk_cap || (ecap && (c.rc[5] > ecap || c.rc[6] > ecap)))
        st = 2;
    else if (nw == 0)
        st = 1;
    else if (k >= cap_iter)
        st = 3;
    out[1] = (unsigned long long)st;
    __threadfence_system();
    if (st) *stop = st;
    if (st == 2) return;   // the host redoes iteration k: keep its tables and its count
    // iteration k+1 reads T_k: swap the pointer tables of the outputs, restart the count
    for (int o = 0; o < n_out; ++o) {
        const int A = out_nt[o];
        uint32_t* t = const_cast<uint32_t*>(Tptr[A]);
        Tptr[A] = Tnptr[A];
        Tnptr[A] = t;
    }
    for (int t = 0; t < n_nt + 2; ++t) new_cells[t] = 0ull;
}

cudaError_t rows_pipe_begin(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, cudaStream_t s) {
    cudaError_t c;
    if (!e->d_stop) {
        if ((c = cudaMalloc(&e->d_stop, sizeof(int))) != cudaSuccess) return c;
        if ((c = cudaHostAlloc(&e->h_map, 32 * sizeof(unsigned long long), cudaHostAllocMapped)) != cudaSuccess) return c;
        if ((c = cudaHostGetDevicePointer(&e->d_map, e->h_map, 0)) != cudaSuccess) return c;
    }
    if ((c = cudaMemsetAsync(e->d_stop, 0, sizeof(int), s)) != cudaSuccess) return c;
    if ((c = dense_set_tables(e, T, Tn, s)) != cudaSuccess) return c;
    if ((c = cudaMemsetAsync(e->new_cells, 0, (e->n_nt + 2) * 8, s)) != cudaSuccess) return c;
    e->pipe = true;
    return cudaSuccess;
}

void rows_pipe_end(DenseEngine* e) { e->pipe = false; }

void rows_set_first(DenseEngine* e, bool first) { e->rows_first = first; }

cudaError_t rows_pipe_clear_stop(DenseEngine* e, cudaStream_t s) {
    return cudaMemsetAsync(e->d_stop, 0, sizeof(int), s);
}

// Upload the T / T_k pointer tables of an iteration (no counter reset).
cudaError_t dense_set_tables(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, cudaStream_t s) {
    cudaError_t c;
    if ((c = cudaMemcpyAsync((void*)e->Tptr, T, e->n_nt * sizeof(void*), cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return c;
    return cudaMemcpyAsync((void*)e->Tnptr, Tn, e->n_nt * sizeof(void*), cudaMemcpyHostToDevice, s);
}

// One iteration, enqueued (gated by the stop flag): rows_begin, rows_shard and the closing
// kernel, which writes the outcome into mapped slot `slot`, swaps the device pointer tables
// and restarts the new-cell count; `done` is recorded behind it.  No host copy per iteration.
cudaError_t rows_pipe_iteration(DenseEngine* e, const NTInfo* nt, const int32_t* adj_idx, const uint64_t* log,
                                unsigned long long n_seeds, bool first, long long k, long long cap_iter, int slot,
                                cudaEvent_t done, cudaStream_t s, int* launches) {
    cudaError_t c;
    e->pipe_enqueue = true;
    c = rows_begin(e, nt, adj_idx, log, n_seeds, first, s, launches);
    if (c == cudaSuccess) c = rows_shard(e, 0, e->n, s, launches);
    e->pipe_enqueue = false;
    if (c != cudaSuccess) return c;
    RowsCtx rc{e->rows_nt, e->rows_adj, e->rcnt, (uint4*)e->dlist, e->dlist_cap, e->rc, 0, 0, 0, e->n, e->l_next,
               e->chunk_cap, 0, 0, e->elist, e->ecap, e->d_stop};
    rows_end_kernel<<<1, 32, 0, s>>>(rc, e->new_cells, e->n_nt, e->chunk_cap, e->elist ? e->ecap : 0, e->d_stop,
                                     e->d_map + 16 * slot, k, cap_iter, e->Tptr, e->Tnptr, e->out_nt, e->n_out);
    if (launches) *launches += 1;
    return cudaEventRecord(done, s);
}

// The outcome of the iteration in `slot` (after its event completed): new cells (~0 = did not
// run), stop reason (0 running, 1 fixpoint, 2 a list ran out, 3 cap), Δ_k words; the chunk
// counters go to h_rc for rows_shard_check.
void rows_pipe_result(DenseEngine* e, int slot, unsigned long long* nw, int* stop, unsigned long long* list_words) {
    volatile unsigned long long* m = e->h_map + 16 * slot;
    *nw = m[0];
    *stop = (int)m[1];
    *list_words = m[2];
    if (*nw != ~0ull)
        for (int q = 0; q < 7; ++q) e->h_rc[q] = m[4 + q];
}

unsigned long long dense_list_capacity(const DenseEngine* e) { return e->dlist_cap; }

bool rows_pipe_eligible(DenseEngine* e) {
    if (e->n_out == 0) return false;
    if (!e->forms_known) {
        for (size_t q = 0; q < e->h_rules.size(); ++q) {
            const bool bc = e->is_const[e->h_rules[q].B], cc = e->is_const[e->h_rules[q].C];
            e->has_r |= bc && !cc;
            e->has_v |= !bc && !cc;
        }
        e->forms_known = true;
    }
    return !e->has_v && e->rgather_variant == 0;
}

// The Δ list ran out during a pipelined run (after a drain): grow it; the next iteration
// rebuilds its T_k buffer by a whole copy.
cudaError_t rows_grow_list(DenseEngine* e, unsigned long long words) {
    if (words <= e->dlist_cap) return cudaSuccess;
    cudaFree(e->dlist);
    e->dlist = nullptr;
    e->dlist_cap = std::max<unsigned long long>(e->dlist_cap * 4, words + words / 4);
    cudaError_t c = cudaMalloc(&e->dlist, e->dlist_cap * sizeof(uint4));
    e->list_complete = false;
    return c;
}

cudaError_t dense_finish(DenseEngine* e, cudaStream_t s, unsigned long long* new_total) {
    cudaError_t c;
    if (!e->h_new && (c = cudaMallocHost(&e->h_new, (e->n_nt + 2) * 8)) != cudaSuccess) return c;
    if ((c = cudaMemcpyAsync(e->h_new, e->new_cells, (e->n_nt + 2) * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return c;
    if ((c = cudaStreamSynchronize(s)) != cudaSuccess) return c;
    *new_total = e->h_new[e->n_nt];
    e->kblocks_total += e->h_new[e->n_nt + 1];
    return cudaSuccess;
}

unsigned long long* dense_total_counter(DenseEngine* e) { return e->new_cells + e->n_nt; }
int64_t dense_row_tiles(const DenseEngine* e) { return e->nt_tiles; }
bool dense_is_fp4(const DenseEngine* e) { return e->fp4; }

// Issued MMA k-blocks (128 x 256 x 128 int8 each) since the last reset.
unsigned long long dense_kblocks(DenseEngine* e, bool reset) {
    unsigned long long v = e->kblocks_total;
    if (reset) e->kblocks_total = 0;
    return v;
}

// ---- Jacobi work accounting (untimed diagnostics): Σ_rules Σ_r |col r of T_B| · |row r of T_C| ----
__global__ void colcount_kernel(const uint32_t* __restrict__ T, int32_t n, int64_t Wp, int32_t rows_per, uint32_t* cnt) {
    int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // column word
    if (w * 32 >= n) return;
    uint32_t c[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) c[b] = 0;
    int r0 = blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
    for (int r = r0; r < r1; ++r) {
        uint32_t v = __ldg(T + (size_t)r * Wp + w);
#pragma unroll
        for (int b = 0; b < 32; ++b) c[b] += (v >> b) & 1u;
    }
#pragma unroll
    for (int b = 0; b < 32; ++b)
        if (c[b] && w * 32 + b < n) atomicAdd(cnt + w * 32 + b, c[b]);
}

__global__ void rowcount_kernel(const uint32_t* __restrict__ T, int32_t n, int64_t Wp, uint32_t* cnt) {
    int lane = threadIdx.x & 31;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n;
         row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t c = 0;
        for (int64_t w = lane; w * 32 < n; w += 32) c += __popc(__ldg(T + (size_t)row * Wp + w));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) cnt[row] = c;
    }
}

__global__ void dot_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int32_t n,
                           unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        acc += (unsigned long long)a[t] * b[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

cudaError_t dense_account(DenseEngine* e, uint32_t* const* T, const std::vector<Rule3>& rules, cudaStream_t s,
                          unsigned long long* out) {
    cudaError_t c;
    if (!e->cnt) {
        if ((c = cudaMalloc(&e->cnt, (size_t)2 * e->n * 4 + 64)) != cudaSuccess) return c;
    }
    uint32_t* colB = e->cnt;
    uint32_t* rowC = e->cnt + e->n;
    unsigned long long* acc = (unsigned long long*)(e->cnt + 2 * (size_t)e->n);
    acc = (unsigned long long*)(((uintptr_t)acc + 7) & ~uintptr_t(7));
    if ((c = cudaMemsetAsync(acc, 0, 8, s)) != cudaSuccess) return c;
    const int rows_per = 1024;
    for (auto& r : rules) {
        if ((c = cudaMemsetAsync(colB, 0, (size_t)e->n * 4, s)) != cudaSuccess) return c;
        dim3 g((unsigned)(((e->n + 31) / 32 + 127) / 128), (unsigned)((e->n + rows_per - 1) / rows_per));
        colcount_kernel<<<g, 128, 0, s>>>(T[r.B], e->n, e->Wp, rows_per, colB);
        rowcount_kernel<<<148 * 8, 256, 0, s>>>(T[r.C], e->n, e->Wp, rowC);
        dot_kernel<<<148 * 4, 256, 0, s>>>(colB, rowC, e->n, acc);
    }
    unsigned long long v = 0;
    if ((c = cudaMemcpyAsync(&v, acc, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return c;
    if ((c = cudaStreamSynchronize(s)) != cudaSuccess) return c;
    *out = v;
    return cudaSuccess;
}

const std::vector<int32_t>& dense_outputs(const DenseEngine* e) { return e->h_out; }

}  // namespace cfpq
