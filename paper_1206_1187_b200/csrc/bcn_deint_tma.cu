// bcn_deint_tma.cu — device deinterleave of wide Interleaved regions as a
// Blackwell tile mover (reference parallel.cpp:81-97, deinterleave).
//
// A wide region (TransposeArgs) is a [rows x width] matrix M[i][w] of 4- or
// 8-byte items at physical slot p0; M[i][w] goes to logical position
// w*wpw + i_base + i. The register-pipelined k_transpose spends most of its
// issue slots on per-item LDG / STS / LDS / STG and stalls on the LSU queue
// (profiles/r02/ncu_deint_registers: lg_throttle / mio_throttle, 13-24% issue,
// 53-66% of DRAM peak). Here the memory movement is done by the TMA engine:
//
//   * loads: 2D tensor maps over the physical region, 128-byte (SWIZZLE_128B)
//     boxes of kCb workers x R/ki rows, S stages in flight per CTA, completion
//     on one mbarrier per stage (expect_tx);
//   * transpose: each thread moves E x E blocks (E = 16 / itemsize) from the
//     input tile to the output tile with 16-byte LDS / STS and a register
//     transpose, conflict-free under the swizzle (thread -> block map below);
//   * stores: 2D tensor maps over the logical output, 128-byte boxes of kCb
//     items x CW/ko workers, bulk-group completion (wait_group.read before
//     the output buffer is reused).
//
// TMA needs 16-byte global strides. A row of the physical region is
// width * itemsize bytes and a worker's output run wpw * itemsize, neither a
// multiple of 16 in general, so both sides are viewed as "super-rows" of
// ki = 16 / gcd(16, width * itemsize) rows (resp. ko workers): stride
// ki * width * itemsize is a multiple of 16, and row i is super-row i / ki at
// column offset (i % ki) * width. A tile then takes ki load boxes per column
// block (one per row parity) and ko store boxes per item block. Unaligned
// region starts become a column offset on a 16-byte aligned base.
//
// TMA covers rows [0, RT) x workers [0, WT) with RT a multiple of the store
// box (kCb items) and WT a multiple of ko: a store box never crosses into
// another worker's run or region. The remaining < kCb rows go through
// k_transpose (as a region of their own) and the < ko last workers through a
// small strip kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "bcn_kernels.cuh"

namespace bcn_b200 {

extern std::atomic<uint64_t> g_launches;

namespace {

constexpr int kTmaRows = 128;     // R: items per tile (rows of the physical region)
constexpr int kTmaColBoxes = 2;   // CB: 128-byte load boxes across a tile
constexpr int kTmaStages = 4;     // S: input tiles in flight per CTA
constexpr int kTmaThreads = 256;

template <typename T>
struct TmaTile {
    static constexpr int E = 16 / static_cast<int>(sizeof(T));    // items per 16-byte vector
    static constexpr int kCb = 128 / static_cast<int>(sizeof(T)); // items per 128-byte box row
    static constexpr int R = kTmaRows;
    static constexpr int CW = kCb * kTmaColBoxes;                  // workers per tile
    static constexpr int kBytes = R * CW * static_cast<int>(sizeof(T));  // 32 KiB
    static constexpr int NBI = R / E, NBW = CW / E;                // E x E blocks
    static constexpr int kBlocksPerThread = NBI * NBW / kTmaThreads;
    static_assert(NBW == 8 * kTmaColBoxes, "8 chunks of 16 bytes per 128-byte row");
    static_assert(NBI * NBW % kTmaThreads == 0, "whole blocks per thread");
};

struct TmaArgs {
    uint64_t ntiles, nrb;   // tiles; row blocks per worker block
    uint32_t order;         // 0: worker blocks vary fastest, 1: row blocks
    uint32_t lg_ki, lg_ko;  // log2 of the super-row factors
    uint32_t m2;            // thread -> block skew (bank-conflict map)
    int32_t xin, xout;      // column offsets of the region starts in the maps
    int32_t width;
    int64_t wpw, i_base;
    uint64_t RT;            // TMA rows
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "BCN_TMA_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra BCN_TMA_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// `map` is the generic address of a __grid_constant__ kernel parameter (the
// descriptor must live in param / const / global space, never in a local copy).
__device__ __forceinline__ void tma_load_2d(void* dst, uint64_t map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(uint64_t map, const void* src, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// E x E register transpose of 16-byte row vectors.
__device__ __forceinline__ void transpose_block(const uint4 (&in)[4], uint4 (&out)[4]) {  // 4-byte items
    out[0] = make_uint4(in[0].x, in[1].x, in[2].x, in[3].x);
    out[1] = make_uint4(in[0].y, in[1].y, in[2].y, in[3].y);
    out[2] = make_uint4(in[0].z, in[1].z, in[2].z, in[3].z);
    out[3] = make_uint4(in[0].w, in[1].w, in[2].w, in[3].w);
}
__device__ __forceinline__ void transpose_block(const uint4 (&in)[2], uint4 (&out)[2]) {  // 8-byte items
    out[0] = make_uint4(in[0].x, in[0].y, in[1].x, in[1].y);
    out[1] = make_uint4(in[0].z, in[0].w, in[1].z, in[1].w);
}

template <typename T>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_transpose_tma(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
                    const TmaArgs a) {
    using G = TmaTile<T>;
    constexpr int E = G::E, R = G::R, CW = G::CW, kCb = G::kCb;
    extern __shared__ unsigned char tma_smem_raw[];
    // SWIZZLE_128B boxes need 1024-byte aligned destinations.
    unsigned char* smem = tma_smem_raw + ((1024u - (smem_u32(tma_smem_raw) & 1023u)) & 1023u);
    unsigned char* in_tiles = smem;                                  // [S][kBytes]
    unsigned char* out_tiles = smem + kTmaStages * G::kBytes;        // [2][kBytes]
    __shared__ __align__(8) uint64_t full[kTmaStages];

    const uint64_t in_desc = reinterpret_cast<uint64_t>(&in_map);
    const uint64_t out_desc = reinterpret_cast<uint64_t>(&out_map);
    const unsigned tid = threadIdx.x;
    const uint32_t ki = 1u << a.lg_ki, ko = 1u << a.lg_ko;
    const uint32_t rows_per_in_box = R >> a.lg_ki, rows_per_out_box = CW >> a.lg_ko;
    const uint64_t ntw = (a.ntiles + a.nrb - 1) / a.nrb;
    auto origin = [&](uint64_t t, uint64_t& w0, uint64_t& i0) {
        if (a.order) {
            w0 = (t / a.nrb) * CW;
            i0 = (t % a.nrb) * R;
        } else {
            w0 = (t % ntw) * CW;
            i0 = (t / ntw) * R;
        }
    };
    auto issue_loads = [&](uint64_t t, int s) {
        uint64_t w0, i0;
        origin(t, w0, i0);
        tma_expect_tx(&full[s], G::kBytes);
        unsigned char* dst = in_tiles + s * G::kBytes;
        for (uint32_t p = 0; p < ki; ++p)
            for (int b = 0; b < kTmaColBoxes; ++b)
                tma_load_2d(dst + (p * kTmaColBoxes + b) * rows_per_in_box * 128, in_desc,
                            a.xin + static_cast<int32_t>(p * a.width + w0 + b * kCb),
                            static_cast<int32_t>(i0 >> a.lg_ki), &full[s]);
    };

    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) tma_mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            const uint64_t t = blockIdx.x + static_cast<uint64_t>(s) * gridDim.x;
            if (t < a.ntiles) issue_loads(t, s);
        }
    }
    const uint32_t in_base = smem_u32(in_tiles), out_base = smem_u32(out_tiles);
    for (uint64_t k = 0;; ++k) {
        const uint64_t t = blockIdx.x + k * gridDim.x;
        if (t >= a.ntiles) break;
        const int s = static_cast<int>(k % kTmaStages);
        const uint32_t ob = static_cast<uint32_t>(k & 1);
        if (tid == 0) bulk_wait_read<1>();  // the stores of tile k-2 have read out_tiles[ob]
        __syncthreads();
        tma_wait(&full[s], static_cast<uint32_t>((k / kTmaStages) & 1));
        const uint32_t src = in_base + s * G::kBytes, dst = out_base + ob * G::kBytes;
#pragma unroll
        for (int it = 0; it < G::kBlocksPerThread; ++it) {
            // Thread -> E x E block: 8 consecutive lanes take the 8 16-byte
            // chunks of one 128-byte row segment (bw), skewed across rows (bi)
            // by m2 so both the swizzled reads and writes of a quarter warp
            // hit distinct chunks (host: tma_skew).
            const uint32_t lin = it * kTmaThreads + tid;
            const uint32_t b8 = lin & 7, aa = lin >> 3;
            const uint32_t bw = (aa % kTmaColBoxes) * 8 + b8;
            const uint32_t rest = aa / kTmaColBoxes;
            const uint32_t bi = (rest & ~7u) + ((rest + a.m2 * b8) & 7);
            uint4 v[E], w[E];
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const uint32_t il = E * bi + r;
                const uint32_t p = il & (ki - 1), sr = il >> a.lg_ki;
                const uint32_t box = p * kTmaColBoxes + (bw >> 3);
                v[r] = lds128(src + (box * rows_per_in_box + sr) * 128 + (((bw & 7) ^ (sr & 7)) << 4));
            }
            transpose_block(v, w);
            constexpr uint32_t kItemBoxes = R / kCb;
#pragma unroll
            for (int c = 0; c < E; ++c) {
                const uint32_t wl = E * bw + c;
                const uint32_t q = wl & (ko - 1), u = wl >> a.lg_ko;
                const uint32_t box = q * kItemBoxes + (bi >> 3);
                sts128(dst + (box * rows_per_out_box + u) * 128 + (((bi & 7) ^ (u & 7)) << 4), w[c]);
            }
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            uint64_t w0, i0;
            origin(t, w0, i0);
            const uint64_t rows_here = a.RT - i0 < static_cast<uint64_t>(R) ? a.RT - i0 : R;
            const uint32_t jboxes = static_cast<uint32_t>(rows_here / kCb);
            const unsigned char* ot = out_tiles + ob * G::kBytes;
            for (uint32_t q = 0; q < ko; ++q)
                for (uint32_t j = 0; j < jboxes; ++j)
                    tma_store_2d(out_desc, ot + (q * (R / kCb) + j) * rows_per_out_box * 128,
                                 a.xout + static_cast<int32_t>(q * a.wpw + a.i_base + i0 + j * kCb),
                                 static_cast<int32_t>(w0 >> a.lg_ko));
            bulk_commit();
            const uint64_t tn = t + static_cast<uint64_t>(kTmaStages) * gridDim.x;
            if (tn < a.ntiles) issue_loads(tn, s);
        }
    }
    if (tid == 0) bulk_wait_all();
}

// Workers [w_lo, width) x rows [0, rows): the < ko workers the store maps
// leave out. Tiny (at most 3 * rows items); one thread per item.
template <typename T>
__global__ void __launch_bounds__(256) k_deint_strip(TransposeArgs a, uint64_t w_lo) {
    const T* in = static_cast<const T*>(a.in);
    T* out = static_cast<T*>(a.out);
    const uint64_t nw = a.width - w_lo, total = nw * a.rows;
    for (uint64_t x = blockIdx.x * 256ull + threadIdx.x; x < total; x += 256ull * gridDim.x) {
        const uint64_t w = w_lo + x / a.rows, i = x % a.rows;
        out[w * a.wpw + a.i_base + i] = in[a.p0 + i * a.width + w];
    }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

uint32_t lg2_factor(uint64_t bytes) {  // log2(16 / gcd(16, bytes))
    uint32_t k = 0;
    while (k < 4 && (bytes << k) % 16 != 0) ++k;
    return k;
}

// Skew of the thread -> block map with the fewest bank conflicts for the
// super-row factors (exhaustive search over the map family):
// conflict-free except ki = E with ko < E (2-way on the writes).
uint32_t tma_skew(int E, uint32_t ki, uint32_t ko) {
    if (ko == static_cast<uint32_t>(E)) return 0;
    if (ki == static_cast<uint32_t>(E)) return (E == 4 && ko == 1) ? 2 : 0;
    return 1;
}

bool encode_2d(CUtensorMap* m, int isz, const void* base, uint64_t d0, uint64_t d1, uint64_t stride_bytes,
               uint32_t b0, uint32_t b1) {
    const cuuint64_t dims[2] = {d0, d1};
    const cuuint64_t strides[1] = {stride_bytes};
    const cuuint32_t box[2] = {b0, b1};
    const cuuint32_t estr[2] = {1, 1};
    return encoder()(m, isz == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                     const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T>
cudaError_t tma_region(const TransposeArgs& a, int sms, cudaStream_t s, bool& used) {
    using G = TmaTile<T>;
    constexpr int isz = static_cast<int>(sizeof(T));
    used = false;
    if (!encoder()) return cudaSuccess;
    const uint32_t lg_ki = lg2_factor(a.width * isz), lg_ko = lg2_factor(a.wpw * isz);
    const uint32_t ki = 1u << lg_ki, ko = 1u << lg_ko;
    const uint64_t RT = a.rows / G::kCb * G::kCb;
    const uint64_t WT = a.width / ko * ko;
    if (RT == 0 || WT == 0) return cudaSuccess;
    // Input map: super-rows of ki physical rows from a 16-byte aligned base.
    const uintptr_t in_addr = reinterpret_cast<uintptr_t>(a.in) + a.p0 * isz;
    const uintptr_t in_base = in_addr & ~static_cast<uintptr_t>(15);
    const uint64_t xin = (in_addr - in_base) / isz;
    const uint64_t in_d0 = xin + ki * a.width, in_d1 = RT / ki;
    // Output map: super-rows of ko worker runs.
    const uintptr_t out_addr = reinterpret_cast<uintptr_t>(a.out);
    const uintptr_t out_base = out_addr & ~static_cast<uintptr_t>(15);
    const uint64_t xout = (out_addr - out_base) / isz;
    const uint64_t out_d0 = xout + ko * a.wpw, out_d1 = WT / ko;
    if ((in_addr - in_base) % isz || (out_addr - out_base) % isz) return cudaSuccess;  // misaligned items
    // Every TMA box must START on a 16-byte boundary (measured: a 2D box at an
    // unaligned inner coordinate is an illegal instruction on sm_100a,
    // tools/c/tma_probe.cu), so each parity's row / run starts must be
    // aligned: only regions whose rows and runs are whole 16-byte chunks
    // qualify (ki = ko = 1 and aligned starts); the rest take k_transpose.
    if (ki != 1 || ko != 1 || xin % G::E || (xout + a.i_base) % G::E) return cudaSuccess;
    const uint64_t lim = (1ull << 31) - 1024;
    if (in_d0 > lim || in_d1 > lim || out_d0 > lim || out_d1 > lim || a.i_base + a.rows > lim) return cudaSuccess;
    CUtensorMap in_map, out_map;
    if (!encode_2d(&in_map, isz, reinterpret_cast<const void*>(in_base), in_d0, in_d1, ki * a.width * isz, G::kCb,
                   G::R / ki) ||
        !encode_2d(&out_map, isz, reinterpret_cast<const void*>(out_base), out_d0, out_d1, ko * a.wpw * isz,
                   G::kCb, G::CW / ko))
        return cudaSuccess;  // not encodable: the caller takes the register kernel
    TmaArgs t{};
    t.nrb = (RT + G::R - 1) / G::R;
    const uint64_t ntw = (WT + G::CW - 1) / G::CW;
    t.ntiles = t.nrb * ntw;
    t.lg_ki = lg_ki;
    t.lg_ko = lg_ko;
    t.m2 = tma_skew(G::E, ki, ko);
    t.xin = static_cast<int32_t>(xin);
    t.xout = static_cast<int32_t>(xout);
    t.width = static_cast<int32_t>(std::min<uint64_t>(a.width, lim));
    t.wpw = static_cast<int64_t>(a.wpw);
    t.i_base = static_cast<int64_t>(a.i_base);
    t.RT = RT;
    const size_t smem = static_cast<size_t>(kTmaStages + 2) * G::kBytes + 1024;
    cudaError_t e = cudaFuncSetAttribute(k_transpose_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const uint64_t grid = std::min<uint64_t>(t.ntiles, static_cast<uint64_t>(sms));
    t.order = t.nrb <= 4 * grid ? 1u : 0u;
    k_transpose_tma<T><<<static_cast<unsigned>(grid), kTmaThreads, smem, s>>>(in_map, out_map, t);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    g_launches.fetch_add(1);
    used = true;
    // The < ko last workers over the TMA rows.
    if (WT < a.width) {
        TransposeArgs b = a;
        b.rows = RT;
        const uint64_t items = (a.width - WT) * RT;
        k_deint_strip<T><<<static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, 4096)), 256, 0, s>>>(b, WT);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        g_launches.fetch_add(1);
    }
    // The < kCb last rows of every worker: a region of their own.
    if (RT < a.rows) {
        TransposeArgs b = a;
        b.p0 = a.p0 + RT * a.width;
        b.rows = a.rows - RT;
        b.i_base = a.i_base + RT;
        e = launch_transpose_registers(b, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_transpose_tma(const TransposeArgs& a, int sms, cudaStream_t s, bool* used) {
    bool u = false;
    const cudaError_t e = a.itemsize == 8 ? tma_region<uint64_t>(a, sms, s, u) : tma_region<uint32_t>(a, sms, s, u);
    *used = u;
    return e;
}

}  // namespace bcn_b200
