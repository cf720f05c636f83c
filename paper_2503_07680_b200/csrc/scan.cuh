// scan.cuh — single-pass device-wide exclusive scan (decoupled look-back).
//
// One read and one write of the payload per element: the HBM floor for a
// scan. Each CTA claims a tile (dynamic index for forward progress), loads
// it striped (coalesced), transposes through shared memory to a blocked
// layout, reduces, publishes its aggregate, looks back over predecessor
// tiles with one warp (32 status words per probe), then scans and stores
// striped again. Values are non-negative counts (< 2^62), packed with a
// 2-bit status in one 64-bit word so a status never tears.
//
//   scan_exclusive<ITEMS>(n, load, store, stream, scratch)
//     load(i)            -> T        element i (i < n)
//     store(i, excl)                 receives the exclusive prefix of i
//   returns nothing; the total can be captured by the store functor (i==n-1).
//   scan_exclusive_v: the same with store(i, excl, x), x = load(i) -- stores
//   that need the element (flags from gathers) do not evaluate it again.
#pragma once

#include "common.cuh"

namespace hbp_b200 {

constexpr u64 kScanFlagAgg = 1ull << 62;
constexpr u64 kScanFlagInc = 2ull << 62;
constexpr u64 kScanValMask = (1ull << 62) - 1;

template <typename T, int BLOCK, int ITEMS, typename Load, typename Store, bool SV = false>
__global__ void __launch_bounds__(BLOCK) k_scan_lookback(i64 n, Load load, Store store, u64* status,
                                                         u32* counter) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    constexpr int TILE = BLOCK * ITEMS;
    T* s_items = reinterpret_cast<T*>(s_dyn);  // [TILE + TILE / 32] padded transpose buffer
    __shared__ T s_red[33];
    __shared__ u32 s_tile;
    __shared__ T s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const i64 tile = s_tile;
    const i64 base = tile * TILE;
    auto pad = [](int i) { return i + (i >> 5); };

    // striped coalesced load -> blocked registers
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int li = k * BLOCK + threadIdx.x;
        const i64 gi = base + li;
        s_items[pad(li)] = gi < n ? load(gi) : T(0);
    }
    __syncthreads();
    T local = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) local += s_items[pad(threadIdx.x * ITEMS + k)];
    T total;
    const T texcl = block_exclusive_scan<T>(local, s_red, total);

    // publish + look back
    if (threadIdx.x == 0) {
        // flag and value travel in one 64-bit word: no fence (no other data
        // of this tile is read by its successors)
        const u64 word = (tile == 0 ? kScanFlagInc : kScanFlagAgg) | (static_cast<u64>(total) & kScanValMask);
        *reinterpret_cast<volatile u64*>(&status[tile]) = word;
    }
    if (tile > 0 && threadIdx.x < 32) {
        T acc = 0;
        i64 look = tile - 1;
        const unsigned lane = threadIdx.x;
        while (true) {
            const i64 idx = look - static_cast<i64>(lane);
            u64 w = 0;
            if (idx >= 0) {
                do {
                    w = *reinterpret_cast<volatile u64*>(&status[idx]);
                } while ((w >> 62) == 0);
            } else {
                w = kScanFlagInc;  // virtual inclusive zero before tile 0
            }
            const unsigned inc_mask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
            // lanes up to and including the first inclusive (lowest lane = nearest)
            const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
            T contrib = (static_cast<int>(lane) <= first_inc && idx >= 0) ? static_cast<T>(w & kScanValMask) : T(0);
            acc += warp_sum(contrib);
            if (inc_mask) break;
            look -= 32;
        }
        if (lane == 0) {
            s_prefix = acc;
            *reinterpret_cast<volatile u64*>(&status[tile]) =
                kScanFlagInc | (static_cast<u64>(acc + total) & kScanValMask);
        }
    }
    if (tile == 0 && threadIdx.x == 0) s_prefix = 0;
    __syncthreads();
    T run = s_prefix + texcl;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {  // in place: each thread owns its blocked items
        const T x = s_items[pad(threadIdx.x * ITEMS + k)];
        s_items[pad(threadIdx.x * ITEMS + k)] = run;
        run += x;
    }
    __syncthreads();
    const T tile_end = s_prefix + total;  // inclusive prefix of the tile's last element
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int li = k * BLOCK + threadIdx.x;
        const i64 gi = base + li;
        if (gi < n) {
            if constexpr (SV) {
                const T e = s_items[pad(li)];
                store(gi, e, static_cast<T>((li + 1 < TILE ? s_items[pad(li + 1)] : tile_end) - e));
            } else {
                store(gi, s_items[pad(li)]);
            }
        }
    }
}

// Scratch for scans: status words + tile counters. Each scan takes a fresh,
// already-zeroed stretch of both; the buffers are zeroed again only when a
// stretch would run past their end (scans on a context's stream run in
// order, so a stretch is never reused while a scan still reads it). One
// memset per many scans instead of two per scan.
struct ScanScratch {
    DevBuf<u64> status;
    DevBuf<u32> counter;
    size_t pos = 0, cpos = 0;
    u64* st = nullptr;
    u32* ctr = nullptr;
    void prepare(i64 tiles, cudaStream_t s) {
        const size_t t = static_cast<size_t>(tiles);
        if (status.n < t) {
            status.alloc(t * 4 > (size_t(1) << 16) ? t * 4 : (size_t(1) << 16), s);
            status.zero();
            pos = 0;
        }
        if (counter.n == 0) {
            counter.alloc(4096, s);
            counter.zero();
            cpos = 0;
        }
        if (pos + t > status.n) {
            status.zero();
            pos = 0;
        }
        if (cpos + 1 > counter.n) {
            counter.zero();
            cpos = 0;
        }
        st = status.p + pos;
        ctr = counter.p + cpos;
        pos += t;
        cpos += 1;
    }
};

constexpr int kScanSmallItems = 8;
constexpr i64 kScanSmallTiles = 296;  // 2 x 148 SMs

template <typename T, int ITEMS = 32, int BLOCK = (sizeof(T) == 4 ? 512 : 256), bool SV = false,
          typename Load, typename Store>
void scan_exclusive_impl(i64 n, Load load, Store store, cudaStream_t stream, ScanScratch& scratch, const char* name,
                         double bytes_per_elem) {
    constexpr int TILE = BLOCK * ITEMS;
    if (n <= 0) return;
    if constexpr (ITEMS > kScanSmallItems) {
        // fewer than two large tiles per SM: quarter-size tiles keep every SM busy
        if (n < static_cast<i64>(TILE) * kScanSmallTiles) {
            scan_exclusive_impl<T, kScanSmallItems, BLOCK, SV>(n, load, store, stream, scratch, name, bytes_per_elem);
            return;
        }
    }
    const i64 tiles = (n + TILE - 1) / TILE;
    scratch.prepare(tiles, stream);
    constexpr int smem = static_cast<int>(sizeof(T)) * (TILE + TILE / 32);
    if (smem > 48 * 1024)
        set_max_dynamic_smem_once(reinterpret_cast<const void*>(k_scan_lookback<T, BLOCK, ITEMS, Load, Store, SV>),
                                  smem);
    LAUNCH_B(name, bytes_per_elem * static_cast<double>(n), (k_scan_lookback<T, BLOCK, ITEMS, Load, Store, SV>),
             static_cast<unsigned>(tiles), BLOCK, smem, stream, n, load, store, scratch.st, scratch.ctr);
}

// Large tiles (64 KB of shared memory): the look-back hands the running
// prefix from tile to tile at a roughly fixed cost per tile, so fewer,
// larger tiles keep it off the bandwidth (tools/micro/scan_micro.cu, B200,
// 10M / 100M elements: u64 2048-element tiles 2.0 / 2.4 TB/s, 8192-element
// tiles 2.8 / 3.8 TB/s; u32 16384-element tiles 2.6 / 3.1 TB/s).
template <typename T, int ITEMS = 32, int BLOCK = (sizeof(T) == 4 ? 512 : 256), typename Load, typename Store>
void scan_exclusive(i64 n, Load load, Store store, cudaStream_t stream, ScanScratch& scratch,
                    const char* name = "scan", double bytes_per_elem = 2.0 * sizeof(T)) {
    scan_exclusive_impl<T, ITEMS, BLOCK, false>(n, load, store, stream, scratch, name, bytes_per_elem);
}

// store(i, excl, x) with x = load(i), read back from the tile in shared memory
template <typename T, int ITEMS = 32, int BLOCK = (sizeof(T) == 4 ? 512 : 256), typename Load, typename Store>
void scan_exclusive_v(i64 n, Load load, Store store, cudaStream_t stream, ScanScratch& scratch,
                      const char* name = "scan", double bytes_per_elem = 2.0 * sizeof(T)) {
    scan_exclusive_impl<T, ITEMS, BLOCK, true>(n, load, store, stream, scratch, name, bytes_per_elem);
}

}  // namespace hbp_b200
