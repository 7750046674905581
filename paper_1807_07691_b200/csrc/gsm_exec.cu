// gsm_exec.cu — the SM-based join chain on the device.
//
// Replaces executor.execute / scan / sm_join / parallel_sm_join /
// cross_product / preallocate (/root/reference/pkg/src/gsmat/executor.py:94-368).
//
// One query = one stream-ordered launch sequence with no host round trip
// between plan steps, captured once per plan as a CUDA graph and replayed:
//   k_init    install the query block from its device image, take look-back
//             epochs, resolve constant-endpoint scans (R2/R3/R5)
//   per step  J1 expand | J2/J3 filter | fused [filter][expand][filter] group |
//             J0 cross | gate  (one kernel each; hub pieces drained by k_drain)
//   pack      projection into a row-major u32 result (or fused into the last
//             join), written to pinned host memory when small (zero-copy)
// followed by one sync that returns the per-step counters (the report and the
// budget checks), then optional DISTINCT and the result hand-off.  A batch of
// independent queries (gsm_execute_batch) is captured as ONE graph forking
// over the queries' contexts.
//
// Every join kernel is a single pass of "count -> scan -> scatter" (the
// paper's Alg. 4 N/P pre-allocation, executor.py:197-215) fused into one
// persistent kernel: blocks take 256-row tiles from an atomic counter, each
// thread computes its row's candidate count (N), the block scans the tile
// and a warp-parallel decoupled look-back yields the tile's output offset
// (P); the same block then scatters the tile's outputs into [P, P+N) by
// degree tier: short rows through a swizzled shared-memory window (coalesced
// stores), rows of >= 32 candidates warp-cooperatively, and hub rows of the
// power-law tail (>= 256) as 1024-output pieces drained by k_drain on every SM.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <utility>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cub/cub.cuh>

#include "gsm_internal.cuh"

namespace gsm {

constexpr int TS_THREADS = 256;
constexpr int TS_ITEMS = 1;
constexpr int TS_TILE = TS_THREADS * TS_ITEMS;
constexpr u64 LB_MASK = (1ull << 40) - 1;
constexpr int WARP_ROW = 32;  // rows with >= this many candidates are written by a warp
constexpr u32 EPOCH_MAX = (1u << 22) - 1;
constexpr size_t ZC_BYTES = (size_t)16 << 10;  // results up to this size are written to host memory directly
constexpr size_t ZC_PACK_BYTES = (size_t)1 << 20;  // ... when k_pack writes them (scan-only plans)

struct TileSync {
  u64* status;            // one word per tile: epoch:22 | flag:2 | value:40
  u32* counter;           // dynamic tile counter (zeroed per query)
  const u32* epoch_ptr;   // this launch's epoch, in the query block (so a captured
                          // CUDA graph replays with fresh epochs and no param change)
  u32 epoch;              // loaded from epoch_ptr at kernel start
};

// Hub rows (>= DEFER_ROW candidates) of an expand are not written by their
// tile's block: they are cut into CHUNK-output pieces and queued, and a
// follow-up kernel (k_drain) spreads the pieces over every SM.
constexpr int DEFER_ROW = 256;
// With many left tiles the blocks already share rows of a few hundred
// candidates, but a single power-law hub (10^4-10^6 candidates) written by
// one warp outlasts the whole kernel (phase trace of chain2 on the 100M
// power-law store: 592 blocks done at 642 us, one hub tile until 881 us):
// such rows are always deferred, and so are all rows >= DEFER_ROW of a tile
// whose total output is far above the expected tile output (>= HEAVY_TILE
// and >= 16x the orientation's average run x tile rows: one tile of that
// store carried ~10^6 outputs, the average ~10^3).  Uniformly heavy tiles
// (LUBM memberOf: ~500 per row everywhere) are not deferred: the queue
// round trip would only add traffic (204 -> 384 us when they were).
constexpr int DEFER_BIG = 8192;
constexpr i64 HEAVY_TILE = 32768;
constexpr int CHUNK = 1024;
struct Chunk {
  i64 r;     // left row
  i64 pos;   // output slot of candidate j0
  u32 aux;   // run begin in dst
  u32 j0;    // first candidate of the piece
  u32 len;   // candidates in the piece
  u32 pad;
};
struct ChunkQueue {
  Chunk* items = nullptr;  // null: deferral disabled
  u32* count = nullptr;    // pieces pushed (zeroed per query)
  u32* head = nullptr;     // pieces taken by k_drain (zeroed per query)
  u32 cap = 0;
  u32 min_len = DEFER_ROW; // rows with at least this many candidates are deferred
  i64 heavy = (i64)1 << 62;  // ... and every row >= DEFER_ROW of a tile with this many outputs
};

// Push row r's candidates [0, c) starting at output pos as CHUNK pieces (one
// warp).  Pieces that do not fit the queue are written by the warp itself.
template <class P>
__device__ void defer_row(const P& p, const DTable& s, const ChunkQueue& q, i64 r, u32 aux, i64 c,
                          i64 pos) {
  const int lane = threadIdx.x & 31;
  const u32 pieces = (u32)((c + CHUNK - 1) / CHUNK);
  u32 base = 0;
  if (lane == 0) base = atomicAdd(q.count, pieces);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (u32 k = lane; k < pieces; k += 32) {
    if (base + k < q.cap) {
      Chunk ch;
      ch.r = r;
      ch.pos = pos + (i64)k * CHUNK;
      ch.aux = aux;
      ch.j0 = k * CHUNK;
      ch.len = (u32)min((i64)CHUNK, c - (i64)k * CHUNK);
      ch.pad = 0;
      q.items[base + k] = ch;
    }
  }
  for (u32 k = (base < q.cap ? q.cap - base : 0); k < pieces; k++) {  // overflow: write here
    const i64 j0 = (i64)k * CHUNK, j1 = min((i64)(k + 1) * CHUNK, c);
    for (i64 j = j0 + lane; j < j1; j += 32) p.emit(s, r, aux, j, pos + j);
  }
}

// The last kernel of a query copies the (then final) step counters to the
// head of the result buffer, so the host reads counters and result rows with
// ONE device->host copy.  "Last block" detection: every block bumps a counter
// after its own counter updates; the block that sees gridDim.x - 1 copies.
//
// Self-cleaning query block (img != null): after the export the same block
// restores the whole query block from the plan's device image and takes the
// next replay's look-back epochs from the context's epoch counter — what
// k_init does at the start of a query, done at the end of the previous one
// instead, so a replay of the same plan on the same context (a prepared
// statement, a repeated batch) needs no k_init launch in front of its joins.
struct ExportArgs {
  const StepStat* src = nullptr;
  StepStat* dst = nullptr;  // null: this kernel is not the query's last
  int n = 0;
  u32* done = nullptr;
  const uint4* img = nullptr;  // self-cleaning: the plan's query-block image
  uint4* blk = nullptr;        // ... the context's query block
  int words16 = 0;
  u32* ctr = nullptr;          // context epoch counter
  u32* epochs = nullptr;       // the block's epoch slots
  int n_epochs = 0;
};
__device__ __forceinline__ void export_if_last(const ExportArgs& x) {
  if (!x.dst) return;
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (gridDim.x == 1) {
      s_last = true;  // the only block is the last (its writes are ordered by the barrier)
    } else {
      __threadfence();
      s_last = atomicAdd(x.done, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const volatile i64* src = reinterpret_cast<const volatile i64*>(x.src);
    i64* dst = reinterpret_cast<i64*>(x.dst);
    if (!x.img) {
      for (int i = threadIdx.x; i < x.n * 4; i += blockDim.x) dst[i] = src[i];
      return;
    }
    // Self-cleaning: the first image words, the epoch counter and the
    // counters to export are loaded together (one round trip, not three);
    // the block is reset only after every counter has been read.
    constexpr int IMG_REG = 4;
    uint4 im[IMG_REG];
#pragma unroll
    for (int k = 0; k < IMG_REG; k++) {
      const int w = threadIdx.x + k * blockDim.x;
      if (w < x.words16) im[k] = x.img[w];
    }
    const u32 base = (threadIdx.x == 0 && x.n_epochs > 0) ? *x.ctr : 0u;
    for (int i = threadIdx.x; i < x.n * 4; i += blockDim.x) dst[i] = src[i];
    __syncthreads();  // the counters are exported before the block is reset
#pragma unroll
    for (int k = 0; k < IMG_REG; k++) {
      const int w = threadIdx.x + k * blockDim.x;
      if (w < x.words16) x.blk[w] = im[k];
    }
    for (int w = threadIdx.x + IMG_REG * blockDim.x; w < x.words16; w += blockDim.x) x.blk[w] = x.img[w];
    __syncthreads();  // the image's epoch slots are overwritten below
    if (threadIdx.x == 0 && x.n_epochs > 0) {
      for (int e = 0; e < x.n_epochs; e++) x.epochs[e] = base + 1 + (u32)e;
      *x.ctr = base + (u32)x.n_epochs;
    }
  }
}

// Look-back status words are self-contained (epoch | flag | value in one
// 64-bit word) and nothing else is published with them, so relaxed
// gpu-scope accesses suffice: a release store would put a MEMBAR.ALL.GPU on
// every tile's critical path (ncu: the top stall of the LUBM join kernels) and
// an acquire load a CCTL.IVALL that drops the whole L1.
__device__ __forceinline__ void st_status_u64(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_status_u64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 lb_word(u32 epoch, u32 flag, i64 v) {
  u64 x = v < 0 ? 0 : (u64)v;
  if (x > LB_MASK) x = LB_MASK;
  return ((u64)epoch << 42) | ((u64)flag << 40) | x;
}

// Decoupled look-back, executed by warp 0 of the block: each round inspects
// the 32 preceding tiles at once (ballot for the nearest inclusive prefix,
// warp-sum of the aggregates in between), so a tile never walks its
// predecessors one dependent load at a time.  Returns the exclusive prefix.
__device__ i64 lookback_warp(const TileSync& ts, u32 t, i64 agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) st_status_u64(ts.status, lb_word(ts.epoch, 2, agg));
    return 0;
  }
  if (lane == 0) st_status_u64(ts.status + t, lb_word(ts.epoch, 1, agg));
  i64 excl = 0;
  i64 top = (i64)t - 1;  // highest predecessor of this window
  for (;;) {
    const i64 j = top - lane;
    u64 w;
    u32 fl;
    if (j >= 0) {
      do {
        w = ld_status_u64(ts.status + j);
        fl = ((u32)(w >> 42) == ts.epoch) ? (u32)(w >> 40) & 3u : 0u;
      } while (fl == 0);
    } else {
      w = 0;
      fl = 2;  // before tile 0: an inclusive prefix of 0
    }
    const u32 pmask = __ballot_sync(0xffffffffu, fl == 2);
    const int first = pmask ? __ffs(pmask) - 1 : 32;  // nearest inclusive prefix
    i64 v = (lane <= first && j >= 0) ? (i64)(w & LB_MASK) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (pmask) break;
    top -= 32;
  }
  if (lane == 0) st_status_u64(ts.status + t, lb_word(ts.epoch, 2, excl + agg));
  return excl;
}

// Block-wide decoupled look-back: all TS_THREADS threads inspect one
// predecessor each per round (256 tiles per round instead of 32), since the
// whole block waits for the tile offset anyway.  The tile's aggregate must
// already be published (lb_publish).  Returns the exclusive prefix (to every
// thread) and publishes the inclusive prefix.
struct LBShared {
  int first[TS_THREADS / 32];
  i64 sum[TS_THREADS / 32];
};
__device__ __forceinline__ void lb_publish(const TileSync& ts, u32 t, i64 agg) {
  if (threadIdx.x == 0) st_status_u64(ts.status + t, lb_word(ts.epoch, t == 0 ? 2 : 1, agg));
}
__device__ i64 lookback_block(const TileSync& ts, u32 t, i64 agg, LBShared& sh) {
  if (t == 0) return 0;  // tile 0 published its inclusive prefix in lb_publish
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = TS_THREADS / 32;
  i64 excl = 0;
  i64 top = (i64)t - 1;
  for (;;) {
    const i64 j = top - tid;
    u64 w = 0;
    u32 fl = 2;  // before tile 0: an inclusive prefix of 0
    if (j >= 0) {
      do {
        w = ld_status_u64(ts.status + j);
        fl = ((u32)(w >> 42) == ts.epoch) ? (u32)(w >> 40) & 3u : 0u;
      } while (fl == 0);
    }
    const u32 bal = __ballot_sync(0xffffffffu, fl == 2);
    if (lane == 0) sh.first[warp] = bal ? warp * 32 + __ffs(bal) - 1 : (1 << 30);
    __syncthreads();
    int first = sh.first[0];
#pragma unroll
    for (int i = 1; i < NW; i++) first = min(first, sh.first[i]);
    i64 v = (tid <= first && j >= 0) ? (i64)(w & LB_MASK) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh.sum[warp] = v;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NW; i++) excl += sh.sum[i];
    __syncthreads();  // sh is reused by the next round / the next tile
    if (first < (1 << 30)) break;
    top -= TS_THREADS;
  }
  if (tid == 0) st_status_u64(ts.status + t, lb_word(ts.epoch, 2, excl + agg));
  return excl;
}

// ---------------------------------------------------------------------------
// The fused count/scan/scatter kernel, parameterised by a row policy P:
//   P::prepare(DTable& smem)   copy the input descriptor into shared memory
//   P::rows(smem)              number of input rows (device-resident)
//   P::count(smem, r, aux, e)  candidates of row r (aux: per-row state)
//   P::emit(smem, r, aux, j, g) write candidate j of row r to output slot g
//   P::finish(total)           publish the output row count
//   P::kAccumE                 accumulate e into st->e (filters)
// ---------------------------------------------------------------------------
template <class P, int ITEMS = 1, bool AHEAD = true>
__global__ void __launch_bounds__(TS_THREADS, 4) k_tilescan(P p, TileSync ts, ExportArgs xa) {
  constexpr int TILE = TS_THREADS * ITEMS;  // rows per tile
  // Count-ahead (256-row tiles, NB = 2): a block counts its NEXT tile and
  // publishes that tile's aggregate before it looks back and scatters the
  // current one, so by the time it looks back its predecessors have
  // published theirs (a steady tile spent ~3 µs of ~14 waiting in the
  // look-back, profiles/r02 trace).  512-row tiles keep one buffer (the
  // second would not fit the 48 KB of static shared memory).
  constexpr int NB = AHEAD && (ITEMS == 1 || P::kWindow) ? 2 : 1;
  __shared__ i64 s_pre[NB][TILE + 1];
  __shared__ u32 s_aux[NB][TILE];
  __shared__ i64 s_wsum[TS_THREADS / 32];
  __shared__ LBShared s_lb;
  __shared__ u32 s_tile;
  __shared__ int s_long[TILE];
  __shared__ int s_nlong;
  __shared__ DTable s_in;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  pdl_wait();  // everything below reads the previous kernel's output
  pdl_trigger();
  ts.epoch = *ts.epoch_ptr;
  // Tiles come from an atomic counter in the order blocks get to them (a
  // static first tile per block — tile b for block b — was 4% slower on the
  // long-row expands: a late-starting block then holds back its successors'
  // look-back); the first grab overlaps the descriptor load.
  if (tid == 0) s_tile = atomicAdd(ts.counter, 1u);
  p.prepare(s_in);
  u32 wtag = 0;  // load-balanced scatter: round tag of the row-start marks
  if constexpr (P::kWindow) P::window_init();
  trace_at(0, 0);
  __syncthreads();
  const i64 n = p.rows(s_in);
  int it = 0;
  const i64 ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 0 && blockIdx.x == 0 && tid == 0) p.finish(0);
  i64 e_acc = 0;

  // count tile t into buffer bf: per-row counts -> exclusive prefix in
  // s_pre[bf] (total at [TILE]), per-row state in s_aux[bf], the left
  // columns staged for the window; then publish the tile's aggregate
  auto count_tile = [&](u32 t, int bf) {
    trace_at(it, 1);
    const i64 base = (i64)t * TILE;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      const int rl = i * TS_THREADS + tid;
      const i64 r = base + rl;
      u32 aux = 0, c = 0;
      if constexpr (P::kWindow) {
        // the tile's left columns, for the load-balanced scatter (issued
        // before the count's dependent lookups so the loads overlap)
        constexpr int WA = P::template win_a<TILE, NB>();
        u32 lv[WA];
        const int na = r < n ? p.template staged_cols<TILE, NB>() : 0;
#pragma unroll
        for (int cc = 0; cc < WA; cc++)
          if (cc < na) lv[cc] = __ldg(s_in.col[cc] + r);
        if (r < n) c = p.count(s_in, r, aux, e_acc);
#pragma unroll
        for (int cc = 0; cc < WA; cc++)
          if (cc < na) P::template left_tiles<TILE, NB>()[bf][cc][rl] = lv[cc];
      } else {
        if (r < n) c = p.count(s_in, r, aux, e_acc);
      }
      s_aux[bf][rl] = aux;
      s_pre[bf][rl] = c;
    }
    __syncthreads();
    trace_at(it, 2);
    i64 v[ITEMS], sum = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      v[i] = s_pre[bf][tid * ITEMS + i];
      sum += v[i];
    }
    i64 x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      i64 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    i64 run = x - sum;
    for (int w = 0; w < warp; w++) run += s_wsum[w];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      s_pre[bf][tid * ITEMS + i] = run;
      run += v[i];
    }
    if (tid == TS_THREADS - 1) s_pre[bf][TILE] = run;
    __syncthreads();
    lb_publish(ts, t, s_pre[bf][TILE]);  // successors can start summing right away
    trace_at(it, 3);
  };

  // look back and scatter tile t (counted into buffer bf)
  auto process_tile = [&](u32 t, int bf) {
    const i64 base = (i64)t * TILE;
    const i64 total = s_pre[bf][TILE];
    const i64* pre = s_pre[bf];
    const u32* auxv = s_aux[bf];
    // Tiles whose rows average < WARP_ROW candidates: load-balanced scatter
    // (does its own look-back, overlapped with its first loads).
    if constexpr (P::kWindow) {
      if (total > 0 && total <= (i64)WARP_ROW * TILE && p.template window_ok<TILE, NB>()) {
        const i64 gb = p.template scatter_balanced<TILE>(pre, auxv, total, ts, t, s_lb, wtag, it,
                                                         P::template left_tiles<TILE, NB>()[bf]);
        if ((i64)t == ntiles - 1 && tid == 0) p.finish(gb + total);
        trace_at(it, 5);
        it++;
        __syncthreads();
        return;
      }
    }
    if (tid == 0) s_nlong = 0;
    __syncthreads();
    const i64 gbase = lookback_block(ts, t, total, s_lb);
    trace_at(it, 4);
    // Scatter (thread tid owns tile rows tid, tid + TS_THREADS, ...).  Rows with fewer
    // than WARP_ROW candidates are written by their own thread (consecutive
    // rows are adjacent in the output, so a warp's stores stay dense); longer
    // rows (hubs) are queued and written warp-cooperatively, 32 consecutive
    // outputs per store instruction, unrolled for memory-level parallelism.
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      const int rl = i * TS_THREADS + tid;
      const i64 mine = pre[rl + 1] - pre[rl];
      if (mine > 0 && mine < WARP_ROW) {
        const i64 pos = gbase + pre[rl];
        const u32 aux = auxv[rl];
        for (i64 j = 0; j < mine; j++) p.emit(s_in, base + rl, aux, j, pos + j);
      } else if (mine >= WARP_ROW) {
        s_long[atomicAdd(&s_nlong, 1)] = rl;
      }
    }
    __syncthreads();
    for (int q = warp; q < s_nlong; q += TS_THREADS / 32) {
      const int r = s_long[q];
      const i64 c = pre[r + 1] - pre[r];
      const i64 pos = gbase + pre[r];
      const u32 aux = auxv[r];
      if (P::kDefer && p.dq.items && c >= (total >= p.dq.heavy ? (i64)DEFER_ROW : (i64)p.dq.min_len)) {
        defer_row(p, s_in, p.dq, base + r, aux, c, pos);
        continue;
      }
      if constexpr (P::kWarpEmit) {
        p.emit_row_warp(s_in, base + r, aux, c, pos);
      } else {
        for (i64 j = lane; j < c; j += 4 * 32) {
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const i64 jj = j + 32 * u;
            if (jj < c) p.emit(s_in, base + r, aux, jj, pos + jj);
          }
        }
      }
    }
    if ((i64)t == ntiles - 1 && tid == 0) p.finish(gbase + total);
    trace_at(it, 5);
    it++;
    __syncthreads();
  };

  // the next tile's index (every tile was taken by some block's first grab
  // when ntiles <= gridDim: no atomic)
  auto grab = [&]() -> u32 {
    if (ntiles <= (i64)gridDim.x) return (u32)ntiles;
    if (tid == 0) s_tile = atomicAdd(ts.counter, 1u);
    __syncthreads();
    const u32 t = s_tile;
    __syncthreads();  // s_tile is rewritten by the next grab
    return t;
  };

  u32 t = s_tile;  // the first grab (read after the barrier above)
  __syncthreads();
  if (NB == 2) {
    int bf = 0;
    if ((i64)t < ntiles) count_tile(t, bf);
    while ((i64)t < ntiles) {
      const u32 tn = grab();
      if ((i64)tn < ntiles) count_tile(tn, bf ^ 1);
      process_tile(t, bf);
      t = tn;
      bf ^= 1;
    }
  } else {
    while ((i64)t < ntiles) {
      count_tile(t, 0);
      process_tile(t, 0);
      t = grab();
    }
  }
  trace_at(3, 7);
  if (P::kAccumE) {
#pragma unroll
    for (int o = 16; o; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
    if (lane == 0 && e_acc) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->e), (unsigned long long)e_acc);
  }
  export_if_last(xa);
}

__device__ __forceinline__ void copy_desc(DTable& dst, const DTable* src, int ncols) {
  const int tid = threadIdx.x;
  if (tid == 0) dst.n = src->n;
  if (tid < ncols) dst.col[tid] = src->col[tid];
}

// J1: one shared variable with a two-variable right pattern -> neighbour expand
// (sm_join / parallel_sm_join without secondary variables, executor.py:168-194,
// 218-280).  New column = the other endpoint, read from the CSR/CSC segment.
// Fused final projection: when the join is the plan's last step and there is
// no DISTINCT, emit() writes the projected row straight into the context's
// result buffer (row-major, fz.k columns) instead of the arena, and
// finish() records the result count in the pack stat (pad = 1, or 3 when the
// result outgrew the result buffer and the host must re-run unfused).
struct FusedOut {
  u32* stage = nullptr;  // result rows: staging buffer (device or pinned host alias),
                         // or the join's own arena half (dev); null = not fused
  i64 cap = 0;           // rows that fit
  int k = 0;
  int dev = 0;           // device-resident result (larger than the staging buffer)
  int pj[GSM_MAX_VARS];
  StepStat* pst = nullptr;
  __device__ void finish(i64 total) const {
    pst->rows = total;
    if (dev) {  // like k_pack's device path: overflow -> grow the arena, re-run
      pst->overflow = total > cap;
      pst->pad = 0;
    } else {
      pst->pad = total <= cap ? 1 : 3;
    }
  }
};

struct ExpandP {
  static constexpr bool kAccumE = false;
  static constexpr bool kDefer = true;
  static constexpr bool kWarpEmit = true;
  static constexpr bool kWindow = true;
  ChunkQueue dq;
  const DTable* L;
  Orient R;
  int li, a;
  u32* out;
  i64 cap;
  DTable* O;
  StepStat* st;
  FusedOut fz;
  __device__ void prepare(DTable& s) const { copy_desc(s, L, a); }
  __device__ i64 rows(const DTable& s) const { return s.n; }
  __device__ u32 count(const DTable& s, i64 r, u32& aux, i64&) const {
    const uint2 sg = seg_lookup(R, __ldg(s.col[li] + r));
    aux = sg.x;
    return sg.y;
  }
  __device__ void emit(const DTable& s, i64 r, u32 aux, i64 j, i64 g) const {
    const u32 nv = __ldg(R.dst + aux + j);
    if (fz.stage) {
      if (g >= fz.cap) return;
      u32* o = fz.stage + g * fz.k;
      for (int x = 0; x < fz.k; x++) {
        const int c = fz.pj[x];
        o[x] = c < a ? __ldg(s.col[c] + r) : nv;
      }
      return;
    }
    if (g >= cap) return;
#pragma unroll 4
    for (int c = 0; c < a; c++) out[(i64)c * cap + g] = __ldg(s.col[c] + r);
    out[(i64)a * cap + g] = nv;
  }
  // One warp writes candidates [j0, j0+32) of row r (output slots pos + j).
  // Fused row-major output: the 32 rows x k words are contiguous, so lane l
  // writes words l, l+32, ... of that block, fetching each value by shuffle
  // (the left columns are the same for all 32 rows) -> 128-byte stores.
  __device__ void emit_warp(const DTable& s, i64 r, u32 aux, i64 j0, i64 c, i64 pos) const {
    const int lane = threadIdx.x & 31;
    const i64 j = j0 + lane;
    const u32 nv = j < c ? __ldg(R.dst + aux + j) : 0u;
    if (fz.stage) {
      const int k = fz.k;
      const i64 rows = min((i64)32, c - j0);
      const u32 lv = lane < a ? __ldg(s.col[lane] + r) : 0u;
      const i64 base = pos + j0;  // output slot of candidate j0
      const int words = (int)rows * k;
      for (int w0 = 0; w0 < words; w0 += 32) {
        const int w = w0 + lane;
        const int rr = w < words ? w / k : 0;
        const int src = w < words ? fz.pj[w - rr * k] : 0;
        const u32 v_left = __shfl_sync(0xffffffffu, lv, src < a ? src : 0);
        const u32 v_new = __shfl_sync(0xffffffffu, nv, rr);
        if (w < words && base + rr < fz.cap) fz.stage[base * k + w] = src < a ? v_left : v_new;
      }
      return;
    }
    if (j < c && pos + j < cap) {
      const i64 g = pos + j;
#pragma unroll 4
      for (int cc = 0; cc < a; cc++) out[(i64)cc * cap + g] = __ldg(s.col[cc] + r);
      out[(i64)a * cap + g] = nv;
    }
  }
  // One warp writes the whole candidate run of a long row: U chunks of 32
  // candidates are loaded before any of them is stored (U loads in flight
  // per warp).  For small left arities the row's left values are hoisted into
  // registers and the columns are streamed through precomputed pointers, so a
  // chunk costs little more than its a+1 coalesced stores.
  //
  // Columns are 16-byte aligned (the arena halves are, and cap_for() keeps
  // the column stride a multiple of 4 ids), so after a head of < 4
  // candidates that brings pos + j to a multiple of 4, every lane writes 4
  // consecutive output slots of each column with one 128-bit store (the
  // left columns are the same value 4 times): one store instruction per
  // column per 128 candidates instead of 4.  Each lane loads its 4
  // candidates with 4 scalar loads (the run's start is not 16-byte aligned);
  // the warp's 4 loads together cover 512 contiguous bytes.
  template <int A>
  __device__ void row_warp_cols(const DTable& s, i64 r, u32 aux, i64 c, i64 pos) const {
    constexpr int U = 4;  // quads per lane in flight: 16 loads before the stores
    const int lane = threadIdx.x & 31;
    u32 lv[A > 0 ? A : 1];
#pragma unroll
    for (int cc = 0; cc < A; cc++) lv[cc] = __ldg(s.col[cc] + r);
    const u32* src = R.dst + aux;
    u32* ob = out + pos;  // column cc of output slot pos + j is ob[cc * cap + j]
    const i64 lim = min(c, cap - pos);
    if (lim <= 0) return;
    if ((((uintptr_t)out | (uintptr_t)(cap * 4)) & 15) != 0) {
      // columns not 16-byte aligned (table-level joins size them exactly):
      // 32-bit coalesced stores
      for (i64 j0 = 0; j0 < lim; j0 += 32 * U) {
        u32 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const i64 j = j0 + 32 * u + lane;
          v[u] = j < lim ? __ldg(src + j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          const i64 j = j0 + 32 * u + lane;
          if (j < lim) {
#pragma unroll
            for (int cc = 0; cc < A; cc++) ob[(i64)cc * cap + j] = lv[cc];
            ob[(i64)A * cap + j] = v[u];
          }
        }
      }
      return;
    }
    const int h = (int)min((i64)((4 - (pos & 3)) & 3), lim);  // head: scalar
    if (lane < h) {
#pragma unroll
      for (int cc = 0; cc < A; cc++) ob[(i64)cc * cap + lane] = lv[cc];
      ob[(i64)A * cap + lane] = __ldg(src + lane);
    }
    const u32* s4 = src + h;
    u32* o4 = ob + h;  // 16-byte aligned in every column
    const i64 nq = (lim - h) >> 2;
    for (i64 q0 = 0; q0 < nq; q0 += 32 * U) {
      u32 v[U][4];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const i64 q = q0 + 32 * u + lane;
#pragma unroll
        for (int k = 0; k < 4; k++) v[u][k] = q < nq ? __ldg(s4 + 4 * q + k) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const i64 q = q0 + 32 * u + lane;
        if (q < nq) {
#pragma unroll
          for (int cc = 0; cc < A; cc++)
            *reinterpret_cast<uint4*>(o4 + (i64)cc * cap + 4 * q) = make_uint4(lv[cc], lv[cc], lv[cc], lv[cc]);
          *reinterpret_cast<uint4*>(o4 + (i64)A * cap + 4 * q) =
              make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
        }
      }
    }
    const i64 t0 = h + 4 * nq;  // tail: < 4 candidates, scalar
    if (t0 + lane < lim) {
      const i64 j = t0 + lane;
#pragma unroll
      for (int cc = 0; cc < A; cc++) ob[(i64)cc * cap + j] = lv[cc];
      ob[(i64)A * cap + j] = __ldg(src + j);
    }
  }
  template <int K>
  __device__ void row_warp_fused(const DTable& s, i64 r, u32 aux, i64 c, i64 pos) const {
    // row-major, K words per row: lane l of a 32-row chunk writes words
    // l, l+32, ..., (K-1)*32+l of the chunk; word w is column w % K of row
    // w / K.  The lane's (row, column, value) per word do not depend on the
    // chunk, so they are set up once; U chunks of candidates are loaded
    // before any is stored (as in row_warp_cols: the chunk loop would
    // otherwise wait one memory round trip per 32 candidates).
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    int rr[K];
    u32 val[K];
    bool nw[K];
#pragma unroll
    for (int x = 0; x < K; x++) {
      const int w = x * 32 + lane;
      rr[x] = w / K;
      const int src = fz.pj[w - rr[x] * K];
      nw[x] = src >= a;
      val[x] = src < a ? __ldg(s.col[src] + r) : 0u;
    }
    const u32* dsrc = R.dst + aux;
    for (i64 j0 = 0; j0 < c; j0 += 32 * U) {
      u32 nv[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const i64 j = j0 + 32 * u + lane;
        nv[u] = j < c ? __ldg(dsrc + j) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const i64 jb = j0 + 32 * u;
        if (jb >= c) break;
        const i64 base = pos + jb;
        const int rows = (int)min((i64)32, c - jb);
#pragma unroll
        for (int x = 0; x < K; x++) {
          const u32 nvr = __shfl_sync(0xffffffffu, nv[u], rr[x]);
          if (rr[x] < rows && base + rr[x] < fz.cap) fz.stage[base * K + x * 32 + lane] = nw[x] ? nvr : val[x];
        }
      }
    }
  }
  __device__ void emit_row_warp(const DTable& s, i64 r, u32 aux, i64 c, i64 pos) const {
    if (fz.stage) {
      // (a 4-rows-per-lane variant with 128-bit stores was slower here:
      // memberOf fused 215 -> 267 us — each store instruction then covers
      // 16-byte pieces 16K bytes apart, so every 32-byte sector is written
      // in halves by different instructions; the shuffle form below keeps
      // each instruction on 128 contiguous bytes)
      switch (fz.k) {
        case 1: row_warp_fused<1>(s, r, aux, c, pos); return;
        case 2: row_warp_fused<2>(s, r, aux, c, pos); return;
        case 3: row_warp_fused<3>(s, r, aux, c, pos); return;
        case 4: row_warp_fused<4>(s, r, aux, c, pos); return;
        default: break;
      }
      for (i64 j0 = 0; j0 < c; j0 += 32) {
        const i64 j = j0 + (threadIdx.x & 31);
        emit_chunk_fused(s, r, j < c ? __ldg(R.dst + aux + j) : 0u, j0, c, pos);
      }
      return;
    }
    switch (a) {
      case 1: row_warp_cols<1>(s, r, aux, c, pos); return;
      case 2: row_warp_cols<2>(s, r, aux, c, pos); return;
      case 3: row_warp_cols<3>(s, r, aux, c, pos); return;
      case 4: row_warp_cols<4>(s, r, aux, c, pos); return;
      default: break;
    }
    const int lane = threadIdx.x & 31;  // generic arity
    for (i64 j = lane; j < c; j += 32) {
      if (pos + j >= cap) break;
      const i64 g = pos + j;
      for (int cc = 0; cc < a; cc++) out[(i64)cc * cap + g] = __ldg(s.col[cc] + r);
      out[(i64)a * cap + g] = __ldg(R.dst + aux + j);
    }
  }
  // Tiles of short rows (average < WARP_ROW candidates): load-balanced
  // scatter.  Output slots, not rows, are dealt to threads: in a round over
  // the window [w, w + WIN), slot w + warp*256 + i*32 + lane (i < SLOTS)
  // belongs to thread (warp, lane), so every store instruction covers 32
  // consecutive output slots whatever the row lengths.  A slot's row comes
  // from "row start" marks in shared memory (row+1 written at the slot where
  // each row's output begins, tagged with the round so marks never need
  // clearing): within a 32-slot chunk, a ballot over the marks and one
  // shuffle give every lane its row; the chunk's carry-in row is the previous
  // chunk's last (a binary search for the warp's first chunk).  All SLOTS
  // neighbour loads are issued before any store; the tile's look-back runs
  // while the first round's loads are in flight.  Left values come from the
  // tile's left columns staged in shared memory by the count phase.
  static constexpr int WIN = 2048, WIN_A = 8, SLOTS = WIN / TS_THREADS, MARK_BITS = 10;
  static constexpr u32 TAG_MAX = (1u << (32 - MARK_BITS)) - 1;
  // the tile's left columns staged by the count phase, one buffer per tile
  // in flight (NB = 2: the count-ahead schedule of k_tilescan).  512-row
  // tiles stage 4 columns, in dynamic shared memory (lt_bytes; the static
  // 48 KB would not hold both buffers)
  // (512-row tiles with one buffer keep 8 static columns: left tables wider
  // than 4 columns take that variant)
  template <int TILE, int NB>
  __host__ __device__ static constexpr bool dyn_lt() { return TILE >= 512 && NB == 2; }
  template <int TILE, int NB>
  __host__ __device__ static constexpr int win_a() { return dyn_lt<TILE, NB>() ? 4 : WIN_A; }
  template <int TILE, int NB>
  __host__ __device__ static constexpr size_t lt_bytes() {
    return dyn_lt<TILE, NB>() ? sizeof(u32) * NB * win_a<TILE, NB>() * TILE : 0;
  }
  template <int TILE, int NB>
  __device__ static u32 (*left_tiles())[win_a<TILE, NB>()][TILE] {
    if constexpr (dyn_lt<TILE, NB>()) {
      extern __shared__ __align__(16) unsigned char gsm_dyn_smem[];
      return reinterpret_cast<u32 (*)[win_a<TILE, NB>()][TILE]>(gsm_dyn_smem);
    } else {
      __shared__ u32 lt[NB][win_a<TILE, NB>()][TILE];
      return lt;
    }
  }
  __device__ static u32 (*marks())[WIN] {
    __shared__ u32 mk[2][WIN];
    return mk;
  }
  template <int TILE>
  __device__ static i64* row_src() {  // per row: dst index of output slot 0
    __shared__ i64 rs[TILE];
    return rs;
  }
  __device__ static void window_init() {  // smem is undefined at kernel start
    u32* mk = &marks()[0][0];
    for (int i = threadIdx.x; i < 2 * WIN; i += TS_THREADS) mk[i] = 0;
  }
  template <int TILE, int NB>
  __device__ int staged_cols() const { return a <= win_a<TILE, NB>() ? a : 0; }
  template <int TILE, int NB>
  __device__ bool window_ok() const {
    return a <= win_a<TILE, NB>() && (!fz.stage || (fz.k >= 1 && fz.k <= 4));
  }
  template <int TILE>
  __device__ static int find_row(const i64* pre, i64 slot) {
    int lo = 0, hi = TILE;  // largest lo with pre[lo] <= slot (pre[0] = 0)
#pragma unroll
    for (int it = 1; it < TILE; it <<= 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= slot) lo = mid; else hi = mid;
    }
    return lo;
  }
  // A = left arity for columnar output (0: runtime a); K = fused row-major width (0: columnar)
  template <int A, int K, int TILE>
  __device__ i64 balanced_rounds(const i64* pre, i64 total, const TileSync& ts, u32 t,
                                 LBShared& lb, u32& wtag, int trace_it, u32 (*lt)[TILE]) const {
    static_assert(TILE <= (1 << (MARK_BITS - 1)), "marks hold row+1 in MARK_BITS bits");
    constexpr int ITEMS = TILE / TS_THREADS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const i64* rsrc = row_src<TILE>();
    i64 gbase = 0;
    int q = 0;
    for (i64 w = 0; w < total; w += WIN, q++) {
      if (wtag == TAG_MAX) {  // tag wrap: clear the marks once (uniform branch)
        __syncthreads();
        window_init();
        __syncthreads();
        wtag = 0;
      }
      const u32 tag = ++wtag;
      u32* m = marks()[q & 1];
#pragma unroll
      for (int i = 0; i < ITEMS; i++) {
        const int rl = i * TS_THREADS + tid;
        const i64 p0 = pre[rl];
        if (pre[rl + 1] > p0 && p0 >= w && p0 < w + WIN) m[p0 - w] = (tag << MARK_BITS) | (u32)(rl + 1);
      }
      __syncthreads();
      const int ws = warp * (32 * SLOTS);  // this warp's first slot in the window
      int carry = w + ws < total ? find_row<TILE>(pre, w + ws) : 0;
      int rr[SLOTS];
#pragma unroll
      for (int i = 0; i < SLOTS; i++) {
        const int sl = ws + i * 32 + lane;
        const u32 mv = m[sl];
        const u32 bal = __ballot_sync(0xffffffffu, (mv >> MARK_BITS) == tag);
        const u32 le = bal & (0xffffffffu >> (31 - lane));
        const int srcl = le ? 31 - __clz((int)le) : 0;
        const int rv = (int)(__shfl_sync(0xffffffffu, mv, srcl) & ((1u << MARK_BITS) - 1)) - 1;
        const int row = le ? rv : carry;
        carry = __shfl_sync(0xffffffffu, row, 31);
        rr[i] = w + sl < total ? row : -1;
      }
      u32 nv[SLOTS];
#pragma unroll
      for (int i = 0; i < SLOTS; i++) {
        const i64 slot = w + ws + i * 32 + lane;
        nv[i] = rr[i] >= 0 ? __ldg(R.dst + (rsrc[rr[i]] + slot)) : 0u;
      }
      if (q == 0) {
        gbase = lookback_block(ts, t, total, lb);  // while the loads are in flight
        trace_at(trace_it, 6);
      }
#pragma unroll
      for (int i = 0; i < SLOTS; i++) {
        const i64 g = gbase + w + ws + i * 32 + lane;
        const int r = rr[i];
        if (r < 0) continue;
        if constexpr (K == 0) {
          if (g < cap) {
            if constexpr (A > 0) {
#pragma unroll
              for (int cc = 0; cc < A; cc++) out[(i64)cc * cap + g] = lt[cc][r];
            } else {
              for (int cc = 0; cc < a; cc++) out[(i64)cc * cap + g] = lt[cc][r];
            }
            out[(i64)a * cap + g] = nv[i];
          }
        } else {
          if (g < fz.cap) {
            u32* o = fz.stage + g * K;
#pragma unroll
            for (int x = 0; x < K; x++) {
              const int src = fz.pj[x];
              o[x] = src < a ? lt[src][r] : nv[i];
            }
          }
        }
      }
      if (q == 0) trace_at(trace_it, 7);
    }
    return gbase;
  }
  template <int TILE>
  __device__ i64 scatter_balanced(const i64* pre, const u32* auxv, i64 total, const TileSync& ts,
                                  u32 t, LBShared& lb, u32& wtag, int trace_it,
                                  u32 (*lt)[TILE]) const {
#pragma unroll
    for (int i = 0; i < TILE / TS_THREADS; i++) {  // read after round 0's barrier
      const int rl = i * TS_THREADS + threadIdx.x;
      row_src<TILE>()[rl] = (i64)auxv[rl] - pre[rl];
    }
    if (fz.stage) {
      switch (fz.k) {
        case 1: return balanced_rounds<0, 1, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
        case 2: return balanced_rounds<0, 2, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
        case 3: return balanced_rounds<0, 3, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
        default: return balanced_rounds<0, 4, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
      }
    }
    switch (a) {
      case 1: return balanced_rounds<1, 0, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
      case 2: return balanced_rounds<2, 0, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
      case 3: return balanced_rounds<3, 0, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
      case 4: return balanced_rounds<4, 0, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
      default: return balanced_rounds<0, 0, TILE>(pre, total, ts, t, lb, wtag, trace_it, lt);
    }
  }
  // Fused row-major output of candidates [j0, j0+32) (value nv per lane).
  __device__ void emit_chunk_fused(const DTable& s, i64 r, u32 nv, i64 j0, i64 c, i64 pos) const {
    const int lane = threadIdx.x & 31;
    const int k = fz.k;
    const i64 rows = min((i64)32, c - j0);
    const u32 lv = lane < a ? __ldg(s.col[lane] + r) : 0u;
    const i64 base = pos + j0;
    const int words = (int)rows * k;
    for (int w0 = 0; w0 < words; w0 += 32) {
      const int w = w0 + lane;
      const int rr = w < words ? w / k : 0;
      const int src = w < words ? fz.pj[w - rr * k] : 0;
      const u32 v_left = __shfl_sync(0xffffffffu, lv, src < a ? src : 0);
      const u32 v_new = __shfl_sync(0xffffffffu, nv, rr);
      if (w < words && base + rr < fz.cap) fz.stage[base * k + w] = src < a ? v_left : v_new;
    }
  }
  __device__ void finish(i64 total) const {
    O->n = total < cap ? total : cap;
    st->e = total;
    st->rows = total;
    st->overflow = !fz.stage && total > cap;
    if (fz.stage) fz.finish(total);
  }
};

// J2 / J3: every shared variable is already bound -> membership filter.
//   F_PAIR  (?s p ?o), both shared: (L[li], L[lj]) in M      E = |segment of J[0]|
//   F_CONST (?s p C) / (C p ?o):    (L[li], C) in M           E = kept rows
//   F_SELF  (?x p ?x):              (L[li], L[li]) in M       E = kept rows
enum { F_PAIR = 0, F_CONST = 1, F_SELF = 2 };
struct FilterP {
  static constexpr bool kWindow = false;
  static constexpr bool kWarpEmit = false;
  static constexpr bool kAccumE = true;
  static constexpr bool kDefer = false;
  ChunkQueue dq;
  const DTable* L;
  Orient R;
  int li, lj, a, mode;
  u32 cval;
  u32* out;
  i64 cap;
  DTable* O;
  StepStat* st;
  FusedOut fz;
  __device__ void prepare(DTable& s) const { copy_desc(s, L, a); }
  __device__ i64 rows(const DTable& s) const { return s.n; }
  __device__ u32 count(const DTable& s, i64 r, u32& aux, i64& e) const {
    const u32 key = __ldg(s.col[li] + r);
    const uint2 sg = seg_lookup(R, key);
    const u32 target = mode == F_PAIR ? __ldg(s.col[lj] + r) : mode == F_CONST ? cval : key;
    const u32 keep = sg.y ? (u32)sorted_contains(R.dst + sg.x, sg.y, target) : 0u;
    e += mode == F_PAIR ? (i64)sg.y : (i64)keep;
    aux = 0;
    return keep;
  }
  __device__ void emit(const DTable& s, i64 r, u32, i64, i64 g) const {
    if (fz.stage) {
      if (g >= fz.cap) return;
      u32* o = fz.stage + g * fz.k;
      for (int x = 0; x < fz.k; x++) o[x] = __ldg(s.col[fz.pj[x]] + r);
      return;
    }
    if (g >= cap) return;
#pragma unroll 4
    for (int c = 0; c < a; c++) out[(i64)c * cap + g] = __ldg(s.col[c] + r);
  }
  __device__ void finish(i64 total) const {
    O->n = total < cap ? total : cap;
    st->rows = total;
    st->overflow = !fz.stage && total > cap;
    if (fz.stage) fz.finish(total);
  }
};

// ---------------------------------------------------------------------------
// Fused step group: [filters on the left row] [expand] [filters on each
// candidate] as ONE kernel.  The intermediate tables of the fused steps are
// never materialised, but every fused step still produces its exact
// StepReport counters (rows, prealloc_total E) for the report and the budget
// rules: they are accumulated per block in shared memory and added to the
// step's stats slot at the end.  Rows whose candidate list is long (hubs) are
// counted and emitted warp-cooperatively (ballot compaction keeps the output
// positions of surviving candidates dense and ordered).
// ---------------------------------------------------------------------------
constexpr int MAXF = 8;              // filters on each side of the expand
constexpr u32 FUSE_MAX_FANOUT = 4;   // post-expand filters fuse only below this fan-out
// A fused intersection evaluates every candidate of a row inside the block
// that owns the row: a hub row of 10^5 candidates (each a search of the
// closing run) then runs alone on one SM long after the rest (T4 skew store:
// 17 ms for a 2.9M-row expand).  Above this longest run the expand is
// materialised instead and the filter kernel spreads its rows evenly.
constexpr u32 INTERSECT_MAX_FANOUT = 1u << 14;
// ... and below this average run the materialised expand is cheap and the
// filter kernel's rows-in-parallel lookups beat the fused per-row chain
// (power-law triangle, avg run 2: 1.45 ms unfused vs 1.87 fused; LUBM-1000
// c3, 0.15 candidates per left row: 0.22 vs 0.36; c1, 6.2: 1.07 vs 0.54;
// c8, 36: 0.89 vs 0.45)
constexpr i64 INTERSECT_MIN_AVG = 4;
constexpr int MAXGS = 2 * MAXF + 1;  // steps in a group

struct FSpec {
  Orient R;   // orientation searched
  int mode;   // F_PAIR / F_CONST / F_SELF
  int kc;     // virtual-row column of the lookup key (a = the expanded column)
  int tc;     // F_PAIR: virtual-row column of the target
  u32 cval;   // F_CONST target
  int slot;   // counter slot (step) of this filter
};

struct GroupP {
  const DTable* L;
  int a;             // left arity
  int npre, npost;   // f[0, npre) gate left rows, f[npre, npre+npost) test candidates
  FSpec f[2 * MAXF];
  int has_x;         // an expand step is fused
  Orient X;
  int xk, xslot;
  int nslots;
  int last_slot;     // slot of the group's final step
  StepStat* st[MAXGS];
  ChunkQueue dq;     // hub deferral (only when npost == 0)
  u32* out;          // columnar output (when not fused into the result)
  i64 cap;
  DTable* O;
  FusedOut fz;
};

__device__ __forceinline__ u32 vcol(const DTable& s, int a, int c, i64 r, u32 cand) {
  return c < a ? __ldg(s.col[c] + r) : cand;
}

// Evaluate filter f on virtual row (r, cand); accumulate E / rows into the
// calling thread's private counters when acc (reduced once per kernel).
__device__ __forceinline__ bool gfilter(const FSpec& f, const DTable& s, int a, i64 r, u32 cand,
                                        i64* acc) {
  const u32 key = vcol(s, a, f.kc, r, cand);
  const uint2 sg = seg_lookup(f.R, key);
  const u32 target = f.mode == F_PAIR ? vcol(s, a, f.tc, r, cand) : f.mode == F_CONST ? f.cval : key;
  const bool keep = sg.y && sorted_contains(f.R.dst + sg.x, sg.y, target);
  if (acc) {
    acc[2 * f.slot] += f.mode == F_PAIR ? (i64)sg.y : (i64)keep;
    acc[2 * f.slot + 1] += keep;
  }
  return keep;
}

// A post filter whose lookup key is a LEFT column (kc < a) searches the same
// segment for every candidate of the row: with the target being the
// candidate (F_PAIR, tc == a) the filter is a sorted-run INTERSECTION of the
// expand's run and that segment.  The long-row path looks such segments up
// once per row (HOIST of them, in shared memory) instead of per candidate.
constexpr int HOIST = 2;
__device__ __forceinline__ bool gpost_h(const GroupP& p, const DTable& s, i64 r, u32 cand,
                                        const uint2* rsg, i64* acc) {
  for (int i = p.npre; i < p.npre + p.npost; i++) {
    const FSpec& f = p.f[i];
    const int h = i - p.npre;
    uint2 sg;
    u32 key = 0;
    if (h < HOIST && f.kc < p.a) {
      sg = rsg[h];
    } else {
      key = vcol(s, p.a, f.kc, r, cand);
      sg = seg_lookup(f.R, key);
    }
    if (f.mode == F_SELF && f.kc < p.a) key = __ldg(s.col[f.kc] + r);
    const u32 target = f.mode == F_PAIR ? vcol(s, p.a, f.tc, r, cand) : f.mode == F_CONST ? f.cval : key;
    const bool keep = sg.y && sorted_contains(f.R.dst + sg.x, sg.y, target);
    if (acc) {
      acc[2 * f.slot] += f.mode == F_PAIR ? (i64)sg.y : (i64)keep;
      acc[2 * f.slot + 1] += keep;
    }
    if (!keep) return false;
  }
  return true;
}

__device__ __forceinline__ bool gpost(const GroupP& p, const DTable& s, i64 r, u32 cand,
                                      i64* acc) {
  for (int i = p.npre; i < p.npre + p.npost; i++)
    if (!gfilter(p.f[i], s, p.a, r, cand, acc)) return false;
  return true;
}

// Post filters on the (at most GP_BATCH) candidates of one short row, the
// candidates side by side: every filter's lookups for all live candidates
// are issued before any is consumed, so the row pays one dependent chain per
// filter instead of one per (candidate, filter).  Same per-step counters as
// evaluating gpost candidate by candidate.  Returns the survivor bit mask.
constexpr int GP_BATCH = 4;
constexpr int GSURV = 1024;  // survivors of a tile's long rows kept from the count pass
static_assert(GP_BATCH >= (int)FUSE_MAX_FANOUT, "fused post filters must fit one batch");
__device__ __forceinline__ u32 gpost_batch(const GroupP& p, const DTable& s, i64 r, u32 aux, u32 len,
                                           i64* acc, const uint2* hsg) {
  u32 cand[GP_BATCH];
#pragma unroll
  for (int j = 0; j < GP_BATCH; j++) cand[j] = (u32)j < len ? __ldg(p.X.dst + aux + j) : 0u;
  u32 alive = (1u << len) - 1u;
  for (int i = p.npre; i < p.npre + p.npost && alive; i++) {
    const FSpec& f = p.f[i];
    uint2 sg[GP_BATCH];
    u32 tgt[GP_BATCH];
#pragma unroll
    for (int j = 0; j < GP_BATCH; j++) {
      sg[j] = make_uint2(0u, 0u);
      tgt[j] = 0u;
      if ((alive >> j) & 1u) {
        const u32 key = vcol(s, p.a, f.kc, r, cand[j]);
        // a filter keyed on a left column searches the row's one segment,
        // looked up by the count phase alongside the expand's (hsg)
        sg[j] = (i - p.npre < HOIST && f.kc < p.a) ? hsg[i - p.npre] : seg_lookup(f.R, key);
        tgt[j] = f.mode == F_PAIR ? vcol(s, p.a, f.tc, r, cand[j]) : f.mode == F_CONST ? f.cval : key;
      }
    }
#pragma unroll
    for (int j = 0; j < GP_BATCH; j++) {
      if (!((alive >> j) & 1u)) continue;
      const bool keep = sg[j].y && sorted_contains(f.R.dst + sg[j].x, sg[j].y, tgt[j]);
      acc[2 * f.slot] += f.mode == F_PAIR ? (i64)sg[j].y : (i64)keep;
      acc[2 * f.slot + 1] += keep;
      if (!keep) alive &= ~(1u << j);
    }
  }
  return alive;
}

__device__ __forceinline__ void gwrite(const GroupP& p, const DTable& s, i64 r, u32 cand, i64 g) {
  if (p.fz.stage) {
    if (g >= p.fz.cap) return;
    u32* o = p.fz.stage + g * p.fz.k;
    for (int x = 0; x < p.fz.k; x++) o[x] = vcol(s, p.a, p.fz.pj[x], r, cand);
    return;
  }
  if (g >= p.cap) return;
  for (int c = 0; c < p.a; c++) p.out[(i64)c * p.cap + g] = __ldg(s.col[c] + r);
  if (p.has_x) p.out[(i64)p.a * p.cap + g] = cand;
}

// Emit adaptor of a fused group for deferred hub pieces (no post filters).
struct GroupEmit {
  static constexpr bool kWarpEmit = false;
  GroupP p;
  __device__ void prepare(DTable& s) const { copy_desc(s, p.L, p.a); }
  __device__ void emit(const DTable& s, i64 r, u32 aux, i64 j, i64 g) const {
    gwrite(p, s, r, __ldg(p.X.dst + aux + j), g);
  }
};

__global__ void __launch_bounds__(TS_THREADS, 4) k_group(GroupP p, TileSync ts, ExportArgs xa) {
  __shared__ i64 s_pre[TS_TILE + 1];
  __shared__ u32 s_aux[TS_TILE];
  __shared__ u32 s_len[TS_TILE];
  __shared__ i64 s_wsum[TS_THREADS / 32];
  __shared__ i64 s_base;
  __shared__ u32 s_tile;
  __shared__ int s_long[TS_TILE];
  __shared__ int s_nlong;
  __shared__ DTable s_in;
  // long rows with post filters: flattened candidate prefix, hoisted
  // segments, survivor counts, and the survivors themselves (when they fit)
  __shared__ u32 s_lpre[TS_TILE + 1];
  __shared__ uint2 s_rsg[TS_TILE][HOIST];
  __shared__ u32 s_lcnt[TS_TILE];
  __shared__ uint2 s_surv[GSURV];
  __shared__ u32 s_nsurv;
  __shared__ unsigned char s_bside[TS_TILE];  // long row walks the filter segment (pairx)
  // the group's post filtering is one intersection-shaped pair filter
  const bool pairx = p.npost == 1 && p.f[p.npre].mode == F_PAIR && p.f[p.npre].kc < p.a &&
                     p.f[p.npre].tc == p.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  i64 acc[2 * MAXGS];  // this thread's (E, rows) contribution to each fused step
  for (int k = 0; k < 2 * MAXGS; k++) acc[k] = 0;
  i64* const s_acc = acc;

  pdl_wait();
  pdl_trigger();
  ts.epoch = *ts.epoch_ptr;
  if (tid == 0) {  // the first grab overlaps the descriptor load
    s_tile = atomicAdd(ts.counter, 1u);
    s_nlong = 0;
  }
  copy_desc(s_in, p.L, p.a);
  trace_at(0, 0);
  __syncthreads();
  const i64 n = s_in.n;
  const i64 ntiles = (n + TS_TILE - 1) / TS_TILE;
  int it = 0;
  if (ntiles == 0 && blockIdx.x == 0 && tid == 0) {
    p.O->n = 0;
    if (p.fz.stage) p.fz.finish(0);
  }
  for (bool first = true; ntiles > 0; first = false) {
    if (!first) {
      // every tile was taken by some block's first grab: skip the atomic
      if (ntiles <= (i64)gridDim.x) break;
      if (tid == 0) {
        s_tile = atomicAdd(ts.counter, 1u);
        s_nlong = 0;
      }
      __syncthreads();
    }
    const u32 t = s_tile;
    if ((i64)t >= ntiles) break;
    trace_at(it, 1);
    const i64 base = (i64)t * TS_TILE;
    const i64 r = base + tid;
    // ---- count: pre-filters, expand, post-filters on short candidate lists
    u32 cnt = 0, aux = 0, len = 0, mask = 0xffffffffu;
    bool warp_row = false;
    if (r < n) {
      bool pass = true;
      for (int i = 0; i < p.npre && pass; i++) pass = gfilter(p.f[i], s_in, p.a, r, 0u, s_acc);
      if (pass) {
        if (!p.has_x) {
          len = 1;
          cnt = 1;
        } else {
          // post filters keyed on a left column: their segment lookups go
          // out together with the expand's, not after the candidates
          uint2 hsg[HOIST];
#pragma unroll
          for (int h = 0; h < HOIST; h++) {
            hsg[h] = make_uint2(0u, 0u);
            if (h < p.npost && p.f[p.npre + h].kc < p.a)
              hsg[h] = seg_lookup(p.f[p.npre + h].R, __ldg(s_in.col[p.f[p.npre + h].kc] + r));
          }
          const uint2 sg = seg_lookup(p.X, __ldg(s_in.col[p.xk] + r));
          aux = sg.x;
          len = sg.y;
          acc[2 * p.xslot] += len;
          acc[2 * p.xslot + 1] += len;
          if (len >= WARP_ROW || (p.npost && len > (u32)GP_BATCH)) {
            warp_row = true;  // counted (if filtered) by the block, emitted by a warp / the block
            cnt = p.npost ? 0u : len;
          } else if (p.npost == 0) {
            cnt = len;
          } else if (len <= (u32)GP_BATCH) {
            mask = gpost_batch(p, s_in, r, aux, len, s_acc, hsg);
            cnt = __popc(mask);
          } else {  // (the host fuses post filters only for fan-out <= GP_BATCH)
            mask = 0;
            for (u32 j = 0; j < len; j++)
              if (gpost(p, s_in, r, __ldg(p.X.dst + aux + j), s_acc)) mask |= 1u << j;
            cnt = __popc(mask);
          }
        }
      }
    }
    s_aux[tid] = aux;
    s_len[tid] = len;
    s_pre[tid] = cnt;
    if (warp_row) s_long[atomicAdd(&s_nlong, 1)] = tid;
    __syncthreads();
    const int nlong = s_nlong;
    bool surv_ok = true;
    if (p.npost && nlong) {
      // Block-cooperative counting of the long rows: their candidates form
      // one flattened index space that all 256 threads stride over (a hub
      // row is spread over the whole block, not one warp), with each row's
      // row-invariant filter segments looked up once.  Survivors are kept
      // (row, candidate) in shared memory when they fit, so the emit pass
      // does not evaluate the filters again.
      //
      // A single pair filter keyed on a left column whose target is the
      // candidate is a sorted-run intersection of the expand's run A and the
      // filter's segment B: walk the shorter side and search the other
      // (LUBM-1000 c6: |A| ~ 3,200 alumni of a university, |B| ~ a few
      // advisees).  The filter's counters stay exact: E = |A| x |B| per row
      // (every candidate would have searched B), rows = the survivors.
      u32 myl = 0;
      if (tid < nlong) {
        const int rl = s_long[tid];
        myl = s_len[rl];
        s_lcnt[tid] = 0;
        for (int h = 0; h < HOIST && h < p.npost; h++) {
          const FSpec& f = p.f[p.npre + h];
          if (f.kc < p.a) s_rsg[tid][h] = seg_lookup(f.R, __ldg(s_in.col[f.kc] + base + rl));
        }
        s_bside[tid] = 0;
        if (pairx && s_rsg[tid][0].y < myl) {
          s_bside[tid] = 1;
          acc[2 * p.f[p.npre].slot] += (i64)myl * s_rsg[tid][0].y;
          myl = s_rsg[tid][0].y;
        }
      }
      u32 xs = myl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, xs, o);
        if (lane >= o) xs += y;
      }
      if (lane == 31) s_wsum[warp] = xs;
      if (tid == 0) s_nsurv = 0;
      __syncthreads();
      u32 runl = xs - myl;
      for (int w = 0; w < warp; w++) runl += (u32)s_wsum[w];
      if (tid < nlong) s_lpre[tid] = runl;
      if (tid == nlong - 1) s_lpre[nlong] = runl + myl;
      __syncthreads();
      const u32 tl = s_lpre[nlong];
      for (u32 f = tid; f < tl; f += TS_THREADS) {
        int lo = 0, hi = nlong - 1;  // last q with s_lpre[q] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_lpre[mid] <= f) lo = mid;
          else hi = mid - 1;
        }
        const int rl = s_long[lo];
        u32 cand;
        bool keep;
        if (s_bside[lo]) {  // walk B, search A
          cand = __ldg(p.f[p.npre].R.dst + s_rsg[lo][0].x + (f - s_lpre[lo]));
          keep = sorted_contains(p.X.dst + s_aux[rl], s_len[rl], cand);
          acc[2 * p.f[p.npre].slot + 1] += keep;
        } else {
          cand = __ldg(p.X.dst + s_aux[rl] + (f - s_lpre[lo]));
          keep = gpost_h(p, s_in, base + rl, cand, s_rsg[lo], s_acc);
        }
        if (keep) {
          atomicAdd(&s_lcnt[lo], 1u);
          const u32 k = atomicAdd(&s_nsurv, 1u);
          if (k < GSURV) s_surv[k] = make_uint2((u32)lo, cand);
        }
      }
      __syncthreads();
      if (tid < nlong) s_pre[s_long[tid]] = s_lcnt[tid];
      surv_ok = s_nsurv <= GSURV;
      __syncthreads();
    }
    trace_at(it, 2);
    // ---- block scan of the per-row survivor counts + look-back
    const i64 mine_cnt = s_pre[tid];
    i64 x = mine_cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i64 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    i64 run = x - mine_cnt;
    for (int w = 0; w < warp; w++) run += s_wsum[w];
    s_pre[tid] = run;
    if (tid == TS_THREADS - 1) s_pre[TS_TILE] = run + mine_cnt;
    __syncthreads();
    const i64 total = s_pre[TS_TILE];
    trace_at(it, 3);
    if (warp == 0) {
      const i64 b = lookback_warp(ts, t, total);
      if (lane == 0) s_base = b;
    }
    __syncthreads();
    trace_at(it, 4);
    const i64 gbase = s_base;
    // ---- emit: short rows by their thread, long rows by a warp
    if (!warp_row && mine_cnt > 0) {
      i64 pos = gbase + s_pre[tid];
      if (!p.has_x) {
        gwrite(p, s_in, r, 0u, pos);
      } else {
        for (u32 j = 0; j < len; j++)  // survivors recorded by the count phase
          if ((mask >> j) & 1u) gwrite(p, s_in, r, __ldg(p.X.dst + aux + j), pos++);
      }
    }
    if (p.npost && nlong) {
      // long rows with post filters: positions inside a row by a shared
      // cursor (row order is not contractual), the survivors
      // from the count pass, or -- when they did not fit -- re-evaluated
      if (tid < nlong) s_lcnt[tid] = 0;
      __syncthreads();
      if (surv_ok) {
        for (u32 k = tid; k < s_nsurv; k += TS_THREADS) {
          const uint2 sv = s_surv[k];
          const int rl = s_long[sv.x];
          gwrite(p, s_in, base + rl, sv.y, gbase + s_pre[rl] + atomicAdd(&s_lcnt[sv.x], 1u));
        }
      } else {
        const u32 tl = s_lpre[nlong];
        for (u32 f = tid; f < tl; f += TS_THREADS) {
          int lo = 0, hi = nlong - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_lpre[mid] <= f) lo = mid;
            else hi = mid - 1;
          }
          const int rl = s_long[lo];
          u32 cand;
          bool keep;
          if (s_bside[lo]) {
            cand = __ldg(p.f[p.npre].R.dst + s_rsg[lo][0].x + (f - s_lpre[lo]));
            keep = sorted_contains(p.X.dst + s_aux[rl], s_len[rl], cand);
          } else {
            cand = __ldg(p.X.dst + s_aux[rl] + (f - s_lpre[lo]));
            keep = gpost_h(p, s_in, base + rl, cand, s_rsg[lo], nullptr);
          }
          if (keep) gwrite(p, s_in, base + rl, cand, gbase + s_pre[rl] + atomicAdd(&s_lcnt[lo], 1u));
        }
      }
    }
    for (int q = warp; q < s_nlong && !p.npost; q += TS_THREADS / 32) {
      const int rl = s_long[q];
      const u32 L = s_len[rl], ax = s_aux[rl];
      i64 pos = gbase + s_pre[rl];
      if (p.npost == 0 && p.dq.items && L >= (total >= p.dq.heavy ? (u32)DEFER_ROW : p.dq.min_len)) {
        defer_row(GroupEmit{p}, s_in, p.dq, base + rl, ax, L, pos);
        continue;
      }
      for (u32 j0 = 0; j0 < L; j0 += 32) {
        const u32 j = j0 + lane;
        u32 cand = 0;
        bool ok = false;
        if (j < L) {
          cand = __ldg(p.X.dst + ax + j);
          ok = p.npost == 0 || gpost(p, s_in, base + rl, cand, nullptr);
        }
        const u32 m = __ballot_sync(0xffffffffu, ok);
        if (ok) gwrite(p, s_in, base + rl, cand, pos + __popc(m & ((1u << lane) - 1u)));
        pos += __popc(m);
      }
    }
    if ((i64)t == ntiles - 1 && tid == 0) {
      const i64 tot = gbase + total;
      p.O->n = tot < p.cap ? tot : p.cap;
      p.st[p.last_slot]->overflow = !p.fz.stage && tot > p.cap;
      if (p.fz.stage) p.fz.finish(tot);
    }
    trace_at(it, 5);
    it++;
    __syncthreads();
  }
  trace_at(3, 7);
  // ---- publish the step counters: warp sums, one global atomic per warp
  for (int k = 0; k < p.nslots; k++) {
    i64 e = acc[2 * k], rw = acc[2 * k + 1];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, o);
      rw += __shfl_xor_sync(0xffffffffu, rw, o);
    }
    if (lane == 0) {
      if (e) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st[k]->e), (unsigned long long)e);
      if (rw) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st[k]->rows), (unsigned long long)rw);
    }
  }
  export_if_last(xa);
}

// Drain the hub pieces queued by the preceding expand: blocks grab pieces
// (CHUNK consecutive outputs of one row) until the queue is empty.
template <class E>
__global__ void __launch_bounds__(TS_THREADS, 4) k_drain(E e, ChunkQueue q, ExportArgs xa) {
  __shared__ DTable s_in;
  __shared__ u32 s_idx;
  pdl_wait();
  pdl_trigger();
  e.prepare(s_in);
  __syncthreads();
  const u32 n = min(*q.count, q.cap);
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(q.head, 1u);
    __syncthreads();
    const u32 idx = s_idx;
    if (idx >= n) break;
    const Chunk ch = q.items[idx];
    if constexpr (E::kWarpEmit) {  // each warp writes a 128-candidate slice of the piece
      constexpr u32 SL = CHUNK / (TS_THREADS / 32);
      const u32 w0 = (threadIdx.x >> 5) * SL;
      if (w0 < ch.len)
        e.emit_row_warp(s_in, ch.r, ch.aux + ch.j0 + w0, (i64)min(SL, ch.len - w0), ch.pos + w0);
    } else {
      for (u32 j = threadIdx.x; j < ch.len; j += TS_THREADS)
        e.emit(s_in, ch.r, ch.aux, (i64)ch.j0 + j, ch.pos + j);
    }
    __syncthreads();
  }
  export_if_last(xa);
}

// DISTINCT over packed row-major rows: a row survives iff it wins the CAS
// into an open-addressing set keyed by the whole tuple (executor.py:360-367).
struct DistinctP {
  static constexpr bool kWindow = false;
  static constexpr bool kWarpEmit = false;
  static constexpr bool kAccumE = false;
  static constexpr bool kDefer = false;
  ChunkQueue dq;
  const u32* in;
  const StepStat* nsrc;  // input row count = nsrc->rows (capped by cap_in)
  i64 cap_in;
  int k;
  u32* slots;
  u32 mask;
  u32* out;
  i64 cap_out;
  StepStat* st;
  __device__ void prepare(DTable&) const {}
  __device__ i64 rows(const DTable&) const {
    i64 n = nsrc->rows;
    return n < cap_in ? n : cap_in;
  }
  __device__ u32 count(const DTable&, i64 r, u32& aux, i64&) const {
    const u32* row = in + r * k;
    u32 h = 0x9E3779B9u;
    for (int c = 0; c < k; c++) h = hash32(h ^ row[c]) + (u32)c;
    h &= mask;
    aux = 0;
    for (;;) {
      u32 cur = slots[h];
      if (cur == 0xFFFFFFFFu) {
        u32 prev = atomicCAS(slots + h, 0xFFFFFFFFu, (u32)r);
        if (prev == 0xFFFFFFFFu) return 1u;
        cur = prev;
      }
      const u32* other = in + (i64)cur * k;
      bool eq = true;
      for (int c = 0; c < k && eq; c++) eq = other[c] == row[c];
      if (eq) return 0u;
      h = (h + 1) & mask;
    }
  }
  __device__ void emit(const DTable&, i64 r, u32, i64, i64 g) const {
    if (g >= cap_out) return;
    for (int c = 0; c < k; c++) out[g * k + c] = in[r * k + c];
  }
  __device__ void finish(i64 total) const {
    st->rows = total;
    st->overflow = total > cap_out;
  }
};

// J0: cross product (executor.py:155-165).  Row g = L[g / |R|] ++ R[g % |R|].
// stat: e = |L|, pad = |R| (for the budget message); rows = |L|*|R|.
__global__ void k_cross(const DTable* L, const DTable* R, int a, int b, u32* out, i64 cap,
                        i64 budget, DTable* O, StepStat* st, ExportArgs xa) {
  pdl_wait();
  pdl_trigger();
  const i64 nl = L->n, nr = R->n;
  // |L|*|R| saturated at 2^62 (nl, nr < 2^40 in practice)
  const __int128 t128 = (__int128)nl * (__int128)nr;
  const i64 total = t128 > ((__int128)1 << 62) ? ((i64)1 << 62) : (i64)t128;
  const bool skip = total > budget;  // the host raises ResourceLimitError
  const i64 lim = skip ? 0 : (total < cap ? total : cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    O->n = lim;
    st->e = nl;
    st->pad = nr;
    st->rows = total;
    st->overflow = !skip && total > cap;
  }
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 g = (i64)blockIdx.x * blockDim.x + threadIdx.x; g < lim; g += stride) {
    const i64 i = g / nr, j = g - i * nr;
    for (int c = 0; c < a; c++) out[(i64)c * cap + g] = __ldg(L->col[c] + i);
    for (int c = 0; c < b; c++) out[(i64)(a + c) * cap + g] = __ldg(R->col[c] + j);
  }
  export_if_last(xa);
}

// J0 against a zero-arity right table (a constant-constant pattern, R5):
// the result is the left table itself or nothing -> descriptor aliasing.
__global__ void k_gate(const DTable* L, const DTable* R, int a, DTable* O, StepStat* st,
                       ExportArgs xa) {
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const i64 nl = L->n, nr = R->n;
  if (tid < a) O->col[tid] = L->col[tid];
  if (tid == 0) {
    const i64 total = nr ? nl : 0;
    O->n = total;
    st->e = nl;
    st->pad = nr;
    st->rows = total;
  }
  export_if_last(xa);
}

// Constant-endpoint scans (executor.py:115-126): one thread per job.
enum { J_SEG = 0, J_CONTAINS = 1 };
struct ResolveJob {
  Orient R;
  u32 k1, k2;
  int kind;
  int table;
  int stat;  // step whose rows to record, -1 = none
  int pad;
};
struct ResolveArgs {
  ResolveJob job[GSM_MAX_STEPS];
  int njobs;
};
// First kernel of every query: installs the query block and takes fresh
// look-back epochs, then resolves the constant-endpoint scans (k_resolve's
// jobs).  A replayed graph copies a device-resident image of the block
// (src), so a query needs no host->device copy; src == nullptr when the host
// uploaded the block itself.  Epochs come from a per-context device counter
// that the host mirrors (reserve_epochs), so tile status words never need
// re-zeroing between launches.
__global__ void k_init(const uint4* __restrict__ src, uint4* __restrict__ dst, int words16, u32* ctr,
                       u32* epochs, int n_epochs, ResolveArgs res, DTable* tables, StepStat* stats,
                       DTable* img_tables, StepStat* img_stats) {
  pdl_wait();
  pdl_trigger();
  // The three parts are independent chains of (cold, after an L2 flush)
  // loads; all of them are issued before the block synchronises, so the
  // kernel costs the longest chain, not their sum.  Only the stores into the
  // block wait for the image copy.
  const int i = threadIdx.x;
  u32 base = 0;
  if (i == 0 && n_epochs > 0) base = *ctr;
  uint2 sg = make_uint2(0, 0);
  i64 n = 0;
  if (i < res.njobs) {
    const ResolveJob& jb = res.job[i];
    sg = seg_lookup(jb.R, jb.k1);
    n = jb.kind == J_SEG ? (i64)sg.y : (sg.y && sorted_contains(jb.R.dst + sg.x, sg.y, jb.k2)) ? 1 : 0;
  }
  if (src)
    for (int w = i; w < words16; w += blockDim.x) dst[w] = src[w];
  __syncthreads();
  if (i == 0 && n_epochs > 0) {
    for (int e = 0; e < n_epochs; e++) epochs[e] = base + 1 + (u32)e;
    *ctr = base + (u32)n_epochs;
  }
  if (i >= res.njobs) return;
  const ResolveJob& jb = res.job[i];
  if (jb.kind == J_SEG) tables[jb.table].col[0] = const_cast<u32*>(jb.R.dst) + sg.x;
  tables[jb.table].n = n;
  if (jb.stat >= 0) stats[jb.stat].rows = n;
  // the store is immutable: the resolved scans go into the plan's image too,
  // so self-cleaning replays (no k_init) find them already in the block
  if (img_tables) {
    if (jb.kind == J_SEG) img_tables[jb.table].col[0] = const_cast<u32*>(jb.R.dst) + sg.x;
    img_tables[jb.table].n = n;
    if (jb.stat >= 0) img_stats[jb.stat].rows = n;
  }
}

// Multi-GPU row partitioning of the first table: keep rows [n*i/k, n*(i+1)/k).
__global__ void k_slice(DTable* T, int a, i64 part, i64 parts, StepStat* st) {
  pdl_wait();
  pdl_trigger();
  const i64 n = T->n;
  const i64 lo = (i64)((__int128)n * part / parts), hi = (i64)((__int128)n * (part + 1) / parts);
  __syncthreads();
  if (threadIdx.x < a) T->col[threadIdx.x] += lo;
  __syncthreads();
  if (threadIdx.x == 0) {
    T->n = hi - lo;
    st->rows = hi - lo;
  }
}

// Equal-E row partitioning of the first table ("balanced by
// the count pass's prefix (equal E, not equal L)").  Row r of the first
// table belongs to part own(r) = min(floor(X_r * parts / E), parts - 1),
// X_r = the exclusive prefix of the first join's per-row candidate counts
// N_i (segment lengths), E = their total; part p keeps the contiguous rows
// [B(p), B(p+1)), B(q) = the first row with own >= q.  Row-granular and
// nested: for parts a power of two, own_2P(r) / 2 == own_P(r), so part p of
// P is exactly parts 2p and 2p+1 of 2P (the left-row chunking splits a
// chunk in place on that).  k_slice_sums adds up N_i over SLICE_CHUNKS
// contiguous chunks; k_slice_pick finds, per boundary, the chunk holding it
// from the chunk prefixes, then the row inside that chunk by a block scan of
// its rows.  E = 0 falls back to equal rows (n*p/parts, also nested).
constexpr int SLICE_CHUNKS = 4096;
__device__ __forceinline__ i64 slice_owner(u64 x, u64 E, i64 parts) {
  const i64 o = (i64)((unsigned __int128)x * (u64)parts / E);
  return o < parts - 1 ? o : parts - 1;
}
__global__ void k_slice_sums(const DTable* T, int key, Orient R, u64* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  const i64 n = T->n;
  const i64 nch = n < SLICE_CHUNKS ? n : SLICE_CHUNKS;
  const u32* kc = T->col[key];
  const int lane = threadIdx.x & 31;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 ch = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nch; ch += nw) {
    const i64 lo = (i64)((__int128)n * ch / nch), hi = (i64)((__int128)n * (ch + 1) / nch);
    u64 acc = 0;
    for (i64 r = lo + lane; r < hi; r += 32) acc += seg_lookup(R, __ldg(kc + r)).y;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sums[ch] = acc;
  }
}
__global__ void __launch_bounds__(1024) k_slice_pick(DTable* T, int a, i64 part, i64 parts,
                                                     StepStat* st, const u64* __restrict__ sums,
                                                     int key, Orient R) {
  pdl_wait();
  pdl_trigger();
  constexpr int PER = SLICE_CHUNKS / 1024;
  __shared__ u64 s_w[32];
  __shared__ int s_chunk[2];
  __shared__ u64 s_base[2];
  __shared__ unsigned long long s_row;
  __shared__ u64 s_run;
  const i64 n = T->n;
  const int nch = (int)(n < SLICE_CHUNKS ? n : SLICE_CHUNKS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u64 v[PER], tot = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int ch = tid * PER + i;
    v[i] = ch < nch ? sums[ch] : 0;
    tot += v[i];
  }
  u64 x = tot;  // inclusive warp scan of the per-thread totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  if (tid < 2) {
    s_chunk[tid] = -1;
    s_base[tid] = 0;
  }
  __syncthreads();
  u64 before = x - tot, E = 0;
  for (int w = 0; w < 32; w++) {
    if (w < warp) before += s_w[w];
    E += s_w[w];
  }
  i64 bound[2];
  if (E == 0) {  // no candidates anywhere: equal rows
    bound[0] = (i64)((__int128)n * part / parts);
    bound[1] = (i64)((__int128)n * (part + 1) / parts);
  } else {
    // boundary q in {part, part + 1}: the chunk holding B(q) is the last
    // chunk whose first row's owner is < q (B(0) = 0, B(parts) = n)
#pragma unroll
    for (int i = 0; i < PER; i++) {
      const int ch = tid * PER + i;
      if (ch < nch) {
        const i64 own = slice_owner(before, E, parts);
        const u64 nxt = before + v[i];
        const i64 own_next = ch + 1 < nch ? slice_owner(nxt, E, parts) : parts;
        for (int b = 0; b < 2; b++) {
          const i64 q = part + b;
          if (q > 0 && q < parts && own < q && own_next >= q) {
            s_chunk[b] = ch;
            s_base[b] = before;
          }
        }
      }
      before += v[i];
    }
    __syncthreads();
    for (int b = 0; b < 2; b++) {
      const i64 q = part + b;
      if (q <= 0 || q >= parts) {
        bound[b] = q <= 0 ? 0 : n;
        continue;
      }
      const int ch = s_chunk[b];
      const i64 lo = (i64)((__int128)n * ch / nch), hi = (i64)((__int128)n * (ch + 1) / nch);
      if (tid == 0) {
        s_row = (unsigned long long)hi;  // no row of the chunk qualifies: the next chunk's first
        s_run = s_base[b];
      }
      __syncthreads();
      const u32* kc = T->col[key];
      for (i64 r0 = lo; r0 < hi; r0 += 1024) {
        const i64 r = r0 + tid;
        const u64 c = r < hi ? seg_lookup(R, __ldg(kc + r)).y : 0;
        u64 y = c;  // block-wide inclusive scan of the rows' counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u64 z = __shfl_up_sync(0xffffffffu, y, o);
          if (lane >= o) y += z;
        }
        if (lane == 31) s_w[warp] = y;
        __syncthreads();
        u64 off = 0;
        for (int w = 0; w < warp; w++) off += s_w[w];
        u64 all = 0;
        for (int w = 0; w < 32; w++) all += s_w[w];
        const u64 xr = s_run + off + y - c;  // exclusive prefix of row r
        if (r < hi && slice_owner(xr, E, parts) >= q) atomicMin(&s_row, (unsigned long long)r);
        __syncthreads();
        if (tid == 0) s_run += all;
        __syncthreads();
        if (s_row < (unsigned long long)hi) break;
      }
      bound[b] = (i64)s_row;
      __syncthreads();
    }
  }
  if (tid == 0) {
    const i64 lo = bound[0], hi = bound[1] > bound[0] ? bound[1] : bound[0];
    for (int c = 0; c < a; c++) T->col[c] += lo;
    T->n = hi - lo;
    st->rows = hi - lo;
  }
}

struct ProjArgs {
  int col[GSM_MAX_VARS];
};
// Projection (executor.py:358-359) into row-major u32 rows.  Results that fit
// go to the context's result buffer, whose head the launch sequence copies to
// pinned host memory before its single sync; larger ones go to the arena and
// become a device-resident result.  st->pad = 1 when staged.
__global__ void k_pack(const DTable* T, ProjArgs pj, int k, u32* dev_out, i64 dev_cap,
                       u32* host_out, i64 host_cap, StepStat* st, ExportArgs xa) {
  pdl_wait();
  pdl_trigger();
  i64 n = T->n;
  const bool to_host = host_out != nullptr && n <= host_cap;
  u32* out = to_host ? host_out : dev_out;
  const i64 cap = to_host ? host_cap : dev_cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rows = n;
    st->overflow = n > cap;
    st->pad = to_host;
  }
  if (n > cap) n = cap;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    for (int c = 0; c < k; c++) out[r * k + c] = __ldg(T->col[pj.col[c]] + r);
  export_if_last(xa);
}

// ---------------------------------------------------------------------------
// Table-level joins (gsm_table_join): sm_join / parallel_sm_join /
// cross_product on arbitrary binding tables.
// ---------------------------------------------------------------------------
// Row-major rows -> struct-of-arrays columns (column stride ld >= n).
__global__ void k_rows_to_cols(const u32* __restrict__ rm, i64 n, int a, u32* __restrict__ cols,
                               i64 ld) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n * a; i += stride) {
    const i64 r = i / a, c = i - r * a;
    cols[c * ld + r] = rm[i];
  }
}

// Sort input of the right table's index: (key = first join column, row).
__global__ void k_key_rows(const u32* __restrict__ R, i64 n, int b, int jc, u32* __restrict__ keys,
                           u32* __restrict__ rows) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    keys[i] = R[i * b + jc];
    rows[i] = (u32)i;
  }
}

// Hash index over the runs of a sorted key array, keys stored as key + 1 so
// that 0 stays the empty-slot marker (table ids may be 0).
__global__ void k_hash_runs(const u32* __restrict__ keys, u32 n, u32* __restrict__ slots, u32 mask) {
  const u32 stride = gridDim.x * blockDim.x;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 key = keys[i];
    if (i != 0 && keys[i - 1] == key) continue;
    u32 lo = i, hi = n;  // end of the run
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (keys[mid] <= key) lo = mid + 1; else hi = mid;
    }
    const u32 stored = key + 1u;
    u32 h = hash32(stored) & mask;
    for (;;) {
      const u32 prev = atomicCAS(slots + 4 * h, 0u, stored);
      if (prev == 0u) {
        slots[4 * h + 1] = i;
        slots[4 * h + 2] = lo - i;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// N_i of every left row (preallocate, executor.py:197-215) and E = sum N_i.
__global__ void k_row_counts(const u32* __restrict__ Lk, i64 n, Orient X, i64* __restrict__ cnt,
                             unsigned long long* __restrict__ total) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  unsigned long long acc = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 c = seg_lookup(X, Lk[i]).y;
    cnt[i] = c;
    acc += c;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, acc);
}

// Emitted-row count of a table join without materialising its candidates:
// per left row, the candidates of its first-variable key that agree on every
// further shared variable (executor.py:186-191).  Lets the sequential budget
// rule (executor.py:192-193) trip before E-sized buffers are allocated.
struct SecCols {
  int n;
  int jl[GSM_MAX_VARS], jr[GSM_MAX_VARS];
};
__global__ void k_sec_counts(const u32* __restrict__ Lcols, i64 n, int li, Orient X,
                             const u32* __restrict__ R, int b, SecCols sc,
                             unsigned long long* __restrict__ total) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  unsigned long long acc = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint2 seg = seg_lookup(X, __ldg(Lcols + (i64)li * n + i));
    for (u32 j = 0; j < seg.y; j++) {
      const u32 ri = __ldg(X.dst + seg.x + j);
      bool ok = true;
      for (int k = 0; k < sc.n && ok; k++)
        ok = __ldg(Lcols + (i64)sc.jl[k] * n + i) == __ldg(R + (i64)ri * b + sc.jr[k]);
      acc += ok;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, acc);
}

// Secondary join variables + output gather of the expanded (left ++ right row
// index) table: keep a candidate iff every further shared variable agrees
// (executor.py:186-191); emit left ++ right[rcols] row-major.
struct TFilterP {
  static constexpr bool kWindow = false;
  static constexpr bool kWarpEmit = false;
  static constexpr bool kAccumE = false;
  static constexpr bool kDefer = false;
  ChunkQueue dq;
  const DTable* L;  // a left columns + the right row index at column a
  int a;
  const u32* R;     // right rows, row-major n_right x b
  int b, nsec, nrc;
  int jl[GSM_MAX_VARS], jr[GSM_MAX_VARS], rc[GSM_MAX_VARS];
  u32* out;
  StepStat* st;
  __device__ void prepare(DTable& s) const { copy_desc(s, L, a + 1); }
  __device__ i64 rows(const DTable& s) const { return s.n; }
  __device__ u32 count(const DTable& s, i64 r, u32& aux, i64&) const {
    const u32 ri = __ldg(s.col[a] + r);
    aux = ri;
    for (int i = 0; i < nsec; i++)
      if (__ldg(s.col[jl[i]] + r) != __ldg(R + (i64)ri * b + jr[i])) return 0u;
    return 1u;
  }
  __device__ void emit(const DTable& s, i64 r, u32 aux, i64, i64 g) const {
    const int w = a + nrc;
    u32* o = out + g * w;
    for (int c = 0; c < a; c++) o[c] = __ldg(s.col[c] + r);
    for (int k = 0; k < nrc; k++) o[a + k] = __ldg(R + (i64)aux * b + rc[k]);
  }
  __device__ void finish(i64 total) const { st->rows = total; }
};

// Row-major cross product: row g = L[g / nR] ++ R[g % nR] (executor.py:164).
__global__ void k_cross_rows(const u32* __restrict__ L, i64 nl, int a, const u32* __restrict__ R,
                             i64 nr, int b, u32* __restrict__ out) {
  const i64 total = nl * nr, stride = (i64)gridDim.x * blockDim.x;
  const int w = a + b;
  for (i64 g = (i64)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
    const i64 i = g / nr, j = g - i * nr;
    for (int c = 0; c < a; c++) out[g * w + c] = L[i * a + c];
    for (int c = 0; c < b; c++) out[g * w + a + c] = R[j * b + c];
  }
}

}  // namespace gsm

// ---------------------------------------------------------------------------
// Sharded-mode exchange: group binding rows by the shard
// that owns the next step's key (subject / object id ranges), or by a hash of
// the whole row for a distributed DISTINCT.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 shard_of(const u32* row, int k, int key_col, u64 node_count, u32 parts) {
  if (key_col >= 0) {
    const u32 id = row[key_col];
    if (id == 0 || node_count == 0) return 0;
    const u64 o = ((u64)(id - 1) * parts) / node_count;
    return o < parts ? (u32)o : parts - 1;
  }
  u64 h = 0x9E3779B97F4A7C15ull;
  for (int c = 0; c < k; c++) {
    h ^= row[c];
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  return (u32)(h % parts);
}

__global__ void k_part_count(const u32* __restrict__ rows, i64 n, int k, int key_col, u64 node_count,
                             u32 parts, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int s_hist[];
  for (u32 d = threadIdx.x; d < parts; d += blockDim.x) s_hist[d] = 0;
  __syncthreads();
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    atomicAdd(&s_hist[shard_of(rows + r * k, k, key_col, node_count, parts)], 1u);
  __syncthreads();
  for (u32 d = threadIdx.x; d < parts; d += blockDim.x)
    if (s_hist[d]) atomicAdd(counts + d, (unsigned long long)s_hist[d]);
}

// cursor[d] starts at destination d's first output row; one atomic per
// (warp, destination) via match_any.
__global__ void k_part_scatter(const u32* __restrict__ rows, i64 n, int k, int key_col, u64 node_count,
                               u32 parts, unsigned long long* __restrict__ cursor, u32* __restrict__ out) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (i64 base = (i64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const i64 r = base + threadIdx.x;
    const bool live = r < n;
    const u32 d = live ? shard_of(rows + r * k, k, key_col, node_count, parts) : 0xFFFFFFFFu;
    const u32 peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    unsigned long long pos = 0;
    if (live && lane == leader) pos = atomicAdd(cursor + d, (unsigned long long)__popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(peers & ((1u << lane) - 1));
    if (live)
      for (int c = 0; c < k; c++) out[(i64)pos * k + c] = rows[r * k + c];
  }
}

// ===========================================================================
// Host orchestration
// ===========================================================================
using namespace gsm;

namespace {
// Launch with Programmatic Dependent Launch allowed: the kernel's blocks may
// be scheduled while the previous kernel in the stream drains (they block in
// griddepcontrol.wait until its results are visible), hiding launch latency
// between the dependent steps of a plan.  Captured into graphs as
// programmatic edges.
template <typename... KArgs, typename... Args>
cudaError_t launch_smem(bool pdl, size_t smem, void (*kern)(KArgs...), int grid, int block,
                        cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch(bool pdl, void (*kern)(KArgs...), int grid, int block, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace

namespace {

constexpr int MAX_TABLES = 2 * GSM_MAX_STEPS + 2;
constexpr size_t STAGE_HEAD = 4096;  // >= sizeof(StepStat) * (GSM_MAX_STEPS + 2)
static_assert(sizeof(StepStat) * (GSM_MAX_STEPS + 2) <= STAGE_HEAD, "stage head too small");

// Device query block: everything a query's kernels read/write besides the
// store and the arena.  Uploaded in one H2D copy, read back in one D2H copy.
struct QueryBlock {
  StepStat stats[GSM_MAX_STEPS + 2];
  u32 counters[GSM_MAX_STEPS + 4];
  u32 epochs[GSM_MAX_STEPS + 4];
  u32 qcount[GSM_MAX_STEPS + 4];  // hub-piece queue of each tile-scan launch
  u32 qhead[GSM_MAX_STEPS + 4];
  u32 done[4];  // blocks finished in the query's last kernel (export_if_last)
  DTable tables[MAX_TABLES];
};

enum Home { H_NONE = 0, H_STORE = 1, H_A = 2, H_B = 3 };

enum StepKind { S_SCAN = 0, S_EMPTY, S_EXPAND, S_FILTER, S_CROSS, S_GATE, S_GROUP };

struct StepPlan {
  StepKind kind;
  std::vector<int> schema;
  int out_table = -1;
};

}  // namespace

struct gsm_context {
  gsm_store* store = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  char* arena = nullptr;
  size_t arena_bytes = 0;
  QueryBlock* d_block = nullptr;
  QueryBlock* h_block = nullptr;  // pinned
  u64* d_status = nullptr;
  size_t n_status = 0;
  u32 epoch = 0;
  u32* d_slots = nullptr;
  size_t n_slots = 0;
  Chunk* d_chunks = nullptr;  // hub-piece queue storage (shared by a query's expands)
  u32 chunk_cap = 0;
  int grid_ts = 296;
  cudaEvent_t ev[GSM_MAX_STEPS + 2] = {};
  cudaEvent_t ev_q0 = nullptr, ev_q1 = nullptr;  // whole-query device time
  cudaEvent_t ev_q2 = nullptr;  // end of the (un-captured) DISTINCT tail
  cudaEvent_t ev_b0 = nullptr, ev_b1 = nullptr, ev_done = nullptr;  // batch timing
  // Result staging: [step counters (STAGE_HEAD bytes) | projected rows].
  u32* d_ctr = nullptr;     // device epoch counter (mirrored by `epoch`)
  u64* d_slice = nullptr;   // equal-E partition: per-chunk candidate sums (SLICE_CHUNKS)
  bool use_equal_e = true;  // GSM_EQUAL_ROWS=1: partition the first table by rows
  bool use_intersect = true;  // GSM_NO_INTERSECT=1: no fusion of intersection-shaped filters
  u32* hd_stage = nullptr;  // device alias of h_stage (zero-copy results)
  u32* hd_rows = nullptr;   // = hd_stage + STAGE_HEAD
  u32* h_stage = nullptr;  // pinned host copy
  u32* d_stage = nullptr;  // device buffer written by the query's last kernel(s)
  u32* h_rows = nullptr;   // = h_stage + STAGE_HEAD
  u32* d_rows = nullptr;   // = d_stage + STAGE_HEAD
  size_t stage_bytes = 0;  // capacity for rows
  size_t guess = 0;        // bytes of the result D2H copied inside the launch sequence
  std::unordered_map<std::string, size_t> last_bytes;  // per plan: last result size
  u64 gen = 0;             // bumped by every gsm_execute (staged results expire)
  bool use_graphs = true;  // replay each distinct query's launch sequence as a CUDA graph
  bool use_pdl = true;     // programmatic dependent launch between plan steps
  bool use_fusion = true;  // fuse [filters][expand][filters] step groups into one kernel
  bool use_defer = true;   // spread hub rows over all SMs (k_drain)
  bool use_proj_fusion = true;  // write the projected result from the last join
  bool use_batch_graph = true;  // a repeated batch replays as one graph (gsm_execute_batch)
  bool batch_poll = true;       // complete batch members as their branches finish (GSM_BATCH_POLL=0: one wait)
  bool batch_pdl = false;       // programmatic dependent launch inside batch graphs (GSM_BATCH_PDL=1)
  // Adaptive grids: a plan's persistent grids are sized from host-side upper
  // bounds on its tables' rows until it has run once; then from the rows it
  // actually produced (x2 headroom) and its graph is captured again.  Any
  // grid is correct (blocks take tiles from a counter), but a 592-block grid
  // over 20 tiles pays 592 tile-counter atomics, 592 last-block atomics and
  // SM slots other queries of a batch need (GSM_NO_ROW_HINTS=1: off).
  bool use_row_hints = true;
  bool use_self_clean = true;  // GSM_NO_SELF_CLEAN=1: every replay starts with k_init
  bool batch_order = true;     // GSM_BATCH_ORDER=0: batch members captured in input order
  size_t zc_bytes = ZC_BYTES;  // GSM_ZC_BYTES: zero-copy limit of fused-projection results
  std::unordered_map<std::string, std::vector<i64>> row_hints;  // plan key -> rows per step
  int tile_items = 0;           // expand tile rows per thread: 0 = by size, 1 or 2 (GSM_TILE_ITEMS)
  // post filters also fuse into an expand expected to output at least this
  // many rows (left rows x average run), whatever its fan-out, unless its
  // runs are skewed (longest > 64 x average: hub rows would serialise in the
  // fused kernel) (GSM_FUSE_HUGE)
  i64 fuse_huge = (i64)1 << 25;
  size_t stage_max = (size_t)1 << 30;  // the staging buffer grows up to this (GSM_STAGE_MAX)
  size_t arena_max = ~(size_t)0;       // the arena grows up to this (GSM_ARENA_MAX)
  // A prepared plan: the captured launch sequence plus what the host needs
  // to replay and complete it without re-planning.
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int kernels = 0;
    std::string image;  // query block bytes uploaded by the sequence's H2D
    int n_epochs = 0;   // tile-scan launches (fresh epochs per replay)
    int pack_stat = 0;
    i64 pack_cap = 0;
    u32* pack_out = nullptr;
    bool fused = false;
    i64 h2d = 0;
    bool zc = false;
    char* d_image = nullptr;  // device copy of `image` (k_init's source)
    // Self-cleaning plans (graphs, no DISTINCT tail): the last kernel
    // restores the query block from d_image, so `warm` — the same sequence
    // without k_init — replays while this image is the one installed.
    bool self_clean = false;
    u64 image_id = 0;                  // process-unique id of d_image's contents
    cudaGraphExec_t warm = nullptr;
    std::vector<int> kinds, arities, fused_in;
  };
  std::unordered_map<std::string, GraphEntry> graphs;
  // A prepared batch (gsm_execute_batch with this context first): the launch
  // sequences of several queries on several contexts captured as ONE graph
  // (fork/join over the contexts' streams), so a repeated batch costs one
  // graph launch instead of one per query.  Valid while every member
  // context's buffers are unchanged (bufgen).
  struct BatchEntry {
    cudaGraphExec_t exec = nullptr;
    // The captured graph (kept: the k_init nodes are toggled in `exec` per
    // launch with cudaGraphNodeSetEnabled): member i's k_init node, and
    // whether it is currently enabled.  A self-cleaning member whose context
    // still holds its image (left clean by its previous replay) runs warm.
    cudaGraph_t graph = nullptr;
    std::vector<cudaGraphNode_t> init_node;
    std::vector<char> init_on;
    bool resolved = false;  // k_init ran once: the images hold the resolved scans
    std::vector<u64> bufgens;
    std::vector<GraphEntry> metas;  // per query (exec unused)
  };
  std::unordered_map<std::string, BatchEntry> batches;
  u64 bufgen = 0;  // process-unique; renewed whenever captured pointers change
  cudaEvent_t ev_fork = nullptr;
  // Recorded (as an external event node) at the end of this context's
  // branch of a batch graph: the host completes each query as soon as its
  // own branch is done, while the rest of the batch still runs.
  cudaEvent_t ev_ext = nullptr;
  // image_id of the self-cleaning plan whose image the query block holds
  // (left clean by that plan's last kernel); 0 = unknown / dirty
  u64 installed = 0;
};

namespace gsm {
u64 context_generation(const gsm_context* c) { return c ? c->gen : ~0ull; }
const u32* context_device_rows(const gsm_context* c) { return c ? c->d_rows : nullptr; }
}

namespace {

// Captured graphs embed arena / staging / status pointers: drop them whenever
// one of those buffers is reallocated.
u64 next_bufgen() {
  static std::atomic<u64> g{0};
  return ++g;
}

u64 next_image_id() {
  static std::atomic<u64> g{0};
  return ++g;
}

void free_batch(gsm_context::BatchEntry& b) {
  cudaGraphExecDestroy(b.exec);
  if (b.graph) cudaGraphDestroy(b.graph);
  for (auto& m : b.metas)
    if (m.d_image) cudaFree(m.d_image);
}

void ctx_clear_graphs(gsm_context* c) {
  for (auto& kv : c->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.warm) cudaGraphExecDestroy(kv.second.warm);
    if (kv.second.d_image) cudaFree(kv.second.d_image);
  }
  c->installed = 0;
  c->graphs.clear();
  for (auto& kv : c->batches) free_batch(kv.second);
  c->batches.clear();
  c->bufgen = next_bufgen();
}

gsm_status ctx_set_arena(gsm_context* c, size_t bytes) {
  ctx_clear_graphs(c);
  if (c->arena) {
    cudaFree(c->arena);
    c->arena = nullptr;
  }
  if (c->d_status) {
    cudaFree(c->d_status);
    c->d_status = nullptr;
  }
  bytes = (bytes + 255) & ~(size_t)255;
  c->gen++;  // results left in the old arena expire
  GSM_CUDA(cudaMalloc(&c->arena, bytes));
  c->arena_bytes = bytes;
  size_t half = bytes / 2;
  if (c->d_chunks) cudaFree(c->d_chunks);
  c->chunk_cap = (u32)std::min<size_t>(std::max<size_t>(65536, half / 4 / 512), 1u << 28);
  GSM_CUDA(cudaMalloc(&c->d_chunks, sizeof(Chunk) * (size_t)c->chunk_cap));
  size_t max_rows = std::max<size_t>(half / 4, c->store->max_nnz) + 1;
  c->n_status = max_rows / TS_TILE + 2;
  GSM_CUDA(cudaMalloc(&c->d_status, c->n_status * sizeof(u64)));
  GSM_CUDA(cudaMemset(c->d_status, 0, c->n_status * sizeof(u64)));
  GSM_CUDA(cudaMemset(c->d_ctr, 0, sizeof(u32)));
  c->epoch = 0;
  return GSM_OK;
}

gsm_status ctx_set_stage(gsm_context* c, size_t bytes) {
  ctx_clear_graphs(c);
  if (c->h_stage) {
    cudaFreeHost(c->h_stage);
    cudaFree(c->d_stage);
    c->h_stage = c->d_stage = c->h_rows = c->d_rows = c->hd_stage = c->hd_rows = nullptr;
    c->stage_bytes = 0;
  }
  bytes = (bytes + 4095) & ~(size_t)4095;
  GSM_CUDA(cudaMallocHost(&c->h_stage, bytes + STAGE_HEAD));
  GSM_CUDA(cudaMalloc(&c->d_stage, bytes + STAGE_HEAD));
  // the launch sequence copies a size GUESS of this buffer to the host
  // (valid rows + a tail the host ignores): defined bytes, once
  GSM_CUDA(cudaMemset(c->d_stage, 0, bytes + STAGE_HEAD));
  c->h_rows = c->h_stage + STAGE_HEAD / 4;
  c->d_rows = c->d_stage + STAGE_HEAD / 4;
  GSM_CUDA(cudaHostGetDevicePointer((void**)&c->hd_stage, c->h_stage, 0));
  c->hd_rows = c->hd_stage + STAGE_HEAD / 4;
  c->stage_bytes = bytes;
  return GSM_OK;
}

// Account for `n` epochs that a k_init enqueued next on c->stream will take
// from the device counter; on wrap-around, re-zero the tile status words and
// the counter first (stream-ordered).
void reserve_epochs(gsm_context* c, int n) {
  if (c->epoch + (u32)n > EPOCH_MAX) {
    cudaMemsetAsync(c->d_status, 0, c->n_status * sizeof(u64), c->stream);
    cudaMemsetAsync(c->d_ctr, 0, sizeof(u32), c->stream);
    c->epoch = 0;
  }
  c->epoch += (u32)n;
}

int index_of(const std::vector<int>& v, int x) {
  for (size_t i = 0; i < v.size(); i++)
    if (v[i] == x) return (int)i;
  return -1;
}

// Right-pattern schema (executor.py:101-110).
std::vector<int> pattern_schema(const gsm_pattern& p) {
  bool sv = p.s_var >= 0, ov = p.o_var >= 0;
  if (sv && ov) return p.s_var == p.o_var ? std::vector<int>{p.s_var} : std::vector<int>{p.s_var, p.o_var};
  if (sv) return {p.s_var};
  if (ov) return {p.o_var};
  return {};
}

struct Exec {
  gsm_context* c;
  const gsm_pattern* steps;
  int n;
  QueryBlock* hb;
  std::vector<StepPlan> plan;
  std::vector<Home> home;  // per table
  std::vector<int> arity;  // per table
  std::vector<i64> ub;     // per table: host-side upper bound on rows (grid sizing)
  int ntables = 0;
  ResolveArgs res{};
  size_t half;

  const PredDev* pred(const gsm_pattern& p) const {
    if (p.empty || p.pid < 1 || p.pid > c->store->max_pid) return nullptr;
    const PredDev& d = c->store->preds[p.pid];
    return d.present ? &d : nullptr;
  }
  char* buf(Home h) const { return c->arena + (h == H_B ? half : 0); }
  int new_table(int a, Home h) {
    int t = ntables++;
    home.push_back(h);
    arity.push_back(a);
    ub.push_back((i64)1 << 62);
    DTable& d = hb->tables[t];
    d.n = 0;
    for (int i = 0; i < GSM_MAX_VARS; i++) d.col[i] = nullptr;
    if (h == H_A || h == H_B) {
      i64 cap = cap_for(a);
      for (int i = 0; i < a; i++) d.col[i] = reinterpret_cast<u32*>(buf(h)) + (i64)i * cap;
    }
    return t;
  }
  // column stride: a multiple of 4 ids, so every column is 16-byte aligned
  // (the vectorised writers' 128-bit stores)
  i64 cap_for(int a) const { return a == 0 ? ((i64)1 << 62) : (i64)(half / (4 * (size_t)a)) & ~(i64)3; }
  static Home other(Home h) { return h == H_A ? H_B : H_A; }

  // Zero-copy table for a pattern read as a whole table (first step, or the
  // right side of a cross product).  Returns table index.
  int scan_table(const gsm_pattern& p, int stat) {
    std::vector<int> sch = pattern_schema(p);
    const PredDev* m = pred(p);
    int t = new_table((int)sch.size(), H_STORE);
    DTable& d = hb->tables[t];
    if (!m) {  // R6: empty flag or no matrix -> zero rows, schema kept
      d.n = 0;
      ub[t] = 0;
      if (stat >= 0) hb->stats[stat].rows = 0;
      return t;
    }
    bool sv = p.s_var >= 0, ov = p.o_var >= 0;
    if (sv && ov && p.s_var != p.o_var) {  // R1: so_pairs
      d.n = m->so.nnz;
      d.col[0] = const_cast<u32*>(m->so.src);
      d.col[1] = const_cast<u32*>(m->so.dst);
      if (stat >= 0) hb->stats[stat].rows = d.n;
    } else if (sv && ov) {  // R4: diagonal
      d.n = m->ndiag;
      d.col[0] = const_cast<u32*>(m->diag);
      if (stat >= 0) hb->stats[stat].rows = d.n;
    } else if (sv || ov) {
      // R2 (?s p C): pairs_for_object(C) -> the s values of C's os run;
      // R3 (C p ?o): pairs_for_subject(C) -> the o values of C's so run.
      // Resolved on the host from the aux arrays: a zero-copy descriptor.
      const HostAux& ha = sv ? c->store->aux_os[p.pid] : c->store->aux_so[p.pid];
      const Orient& R = sv ? m->os : m->so;
      u32 b = 0, len = 0;
      ha.find(sv ? p.o_const : p.s_const, b, len);
      d.n = len;
      d.col[0] = const_cast<u32*>(R.dst) + b;
      if (stat >= 0) hb->stats[stat].rows = d.n;
    } else {  // R5 (C p C'): membership, resolved on the device
      ResolveJob& j = res.job[res.njobs++];
      j.table = t;
      j.stat = stat;
      j.kind = J_CONTAINS;
      j.R = m->so;
      j.k1 = p.s_const;
      j.k2 = p.o_const;
      d.n = 1;  // upper bound until k_init resolves the real value
    }
    ub[t] = d.n;
    return t;
  }
  // Rows to size a grid for: table t's upper bound, or (once the plan has
  // run) twice the rows step `step` produced then, whichever is smaller.
  const std::vector<i64>* hint = nullptr;
  i64 hinted(int t, int step) const {
    i64 r = ub[t];
    if (hint && step >= 0 && step < (int)hint->size()) r = std::min(r, 2 * (*hint)[step] + 1);
    return r;
  }
  // Persistent-grid size for a kernel whose input has at most `rows` rows.
  int grid_for_rows(i64 rows, int per_block) const {
    i64 g = (rows + per_block - 1) / per_block;
    if (g < 1) g = 1;
    return (int)std::min<i64>(g, c->grid_ts);
  }
  static i64 sat_mul(i64 x, i64 y) {
    if (x <= 0 || y <= 0) return 0;
    __int128 z = (__int128)x * y;
    return z > ((__int128)1 << 62) ? ((i64)1 << 62) : (i64)z;
  }
};

}  // namespace

extern "C" {

gsm_status gsm_context_create(gsm_store* store, int64_t arena_bytes, gsm_context** out) {
  *out = nullptr;
  if (!store || !store->finalized) return set_error(GSM_ERR_VALUE, "store missing or not finalized");
  GSM_CUDA(cudaSetDevice(store->device));
  gsm_context* c = new gsm_context();
  c->store = store;
  c->device = store->device;
  if (const char* ng = getenv("GSM_NO_GRAPHS")) c->use_graphs = !(ng[0] == '1');
  if (const char* np = getenv("GSM_NO_PDL")) c->use_pdl = !(np[0] == '1');
  if (const char* nf = getenv("GSM_NO_FUSION")) c->use_fusion = !(nf[0] == '1');
  if (const char* nd = getenv("GSM_NO_DEFER")) c->use_defer = !(nd[0] == '1');
  if (const char* npf = getenv("GSM_NO_PROJ_FUSION")) c->use_proj_fusion = !(npf[0] == '1');
  if (const char* nb = getenv("GSM_NO_BATCH_GRAPH")) c->use_batch_graph = !(nb[0] == '1');
  if (const char* bp = getenv("GSM_BATCH_POLL")) c->batch_poll = !(bp[0] == '0');
  if (const char* bq = getenv("GSM_BATCH_PDL")) c->batch_pdl = bq[0] == '1';
  if (const char* rh = getenv("GSM_NO_ROW_HINTS")) c->use_row_hints = !(rh[0] == '1');
  if (const char* sc = getenv("GSM_NO_SELF_CLEAN")) c->use_self_clean = !(sc[0] == '1');
  if (const char* bo = getenv("GSM_BATCH_ORDER")) c->batch_order = bo[0] != '0';
  if (const char* zb = getenv("GSM_ZC_BYTES")) c->zc_bytes = std::min<size_t>(ZC_PACK_BYTES, strtoull(zb, nullptr, 10));
  if (const char* fh = getenv("GSM_FUSE_HUGE")) c->fuse_huge = std::max<i64>(1, atoll(fh));
  if (const char* ti = getenv("GSM_TILE_ITEMS")) c->tile_items = std::min(2, std::max(0, atoi(ti)));
  if (const char* sm = getenv("GSM_STAGE_MAX")) c->stage_max = std::max<size_t>(4096, strtoull(sm, nullptr, 10));
  // cap on the arena (bytes): below it a plan is evaluated in left-row
  // chunks by the host (tests force chunking on small stores with it)
  if (const char* am = getenv("GSM_ARENA_MAX")) c->arena_max = std::max<size_t>(1 << 20, strtoull(am, nullptr, 10));
  auto fail = [&](gsm_status st) {
    gsm_context_free(c);
    return st;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(cuda_error(e, "cudaStreamCreate"));
  if ((e = cudaMalloc(&c->d_ctr, 16)) != cudaSuccess) return fail(cuda_error(e, "cudaMalloc(epoch counter)"));
  if ((e = cudaMalloc(&c->d_slice, sizeof(u64) * SLICE_CHUNKS)) != cudaSuccess)
    return fail(cuda_error(e, "cudaMalloc(slice sums)"));
  c->use_equal_e = !getenv("GSM_EQUAL_ROWS");
  c->use_intersect = !getenv("GSM_NO_INTERSECT");
  if ((e = cudaMemset(c->d_ctr, 0, 16)) != cudaSuccess) return fail(cuda_error(e, "cudaMemset"));
  if ((e = cudaMalloc(&c->d_block, sizeof(QueryBlock))) != cudaSuccess)
    return fail(cuda_error(e, "cudaMalloc(query block)"));
  if ((e = cudaMallocHost(&c->h_block, sizeof(QueryBlock))) != cudaSuccess)
    return fail(cuda_error(e, "cudaMallocHost(query block)"));
  for (auto& ev : c->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail(cuda_error(e, "cudaEventCreate"));
  if ((e = cudaEventCreate(&c->ev_q0)) != cudaSuccess || (e = cudaEventCreate(&c->ev_q1)) != cudaSuccess ||
      (e = cudaEventCreate(&c->ev_q2)) != cudaSuccess || (e = cudaEventCreate(&c->ev_b0)) != cudaSuccess ||
      (e = cudaEventCreate(&c->ev_b1)) != cudaSuccess || (e = cudaEventCreate(&c->ev_done)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_ext, cudaEventDisableTiming)) != cudaSuccess)
    return fail(cuda_error(e, "cudaEventCreate"));
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // Default arena: 16x the store (64 MB .. 4 GB, at most a quarter of the
  // free memory); a query that outgrows it grows it and re-runs, so a small
  // store's context is cheap to create (the reference's test suites build
  // hundreds of tiny stores).  The staging buffer likewise starts at 2 MB
  // and grows with the results.
  const size_t by_store = std::max<size_t>((size_t)64 << 20, (size_t)store->bytes * 16);
  size_t want = arena_bytes > 0 ? (size_t)arena_bytes
                                : std::min<size_t>(std::min<size_t>((size_t)1 << 32, free_b / 4), by_store);
  gsm_status st = ctx_set_arena(c, std::min(want, c->arena_max));
  if (st != GSM_OK) return fail(st);
  st = ctx_set_stage(c, std::min<size_t>((size_t)2 << 20, c->stage_max));
  if (st != GSM_OK) return fail(st);
  int occ = 0;
  // 512-row expand tiles: static + dynamic shared memory above 48 KB
  static const bool smem_opt_in = [] {
    return cudaFuncSetAttribute(k_tilescan<ExpandP, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ExpandP::lt_bytes<2 * TS_THREADS, 2>()) == cudaSuccess;
  }();
  if (!smem_opt_in) return fail(set_error(GSM_ERR_CUDA, "cudaFuncSetAttribute(k_tilescan<ExpandP, 2>)"));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tilescan<ExpandP>, TS_THREADS, 0);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  c->grid_ts = sms * std::max(1, std::min(occ, 4));
  // (tests: a tiny grid makes every block walk many tiles — the count-ahead
  // schedule and cross-block look-back on small stores)
  if (const char* gm = getenv("GSM_GRID_MAX")) c->grid_ts = std::max(1, std::min(c->grid_ts, atoi(gm)));
  *out = c;
  return GSM_OK;
}

gsm_status gsm_context_capacity(gsm_context* c, int64_t* bytes) {
  if (!c || !bytes) return set_error(GSM_ERR_VALUE, "null context or output");
  GSM_CUDA(cudaSetDevice(c->device));
  size_t free_b = 0, total_b = 0;
  GSM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  size_t avail = free_b + c->arena_bytes;
  if (c->arena_max != ~(size_t)0) avail = std::min(avail, c->arena_max / 9 * 10);
  *bytes = (int64_t)((avail * 9) / 10);
  return GSM_OK;
}

gsm_status gsm_context_stream(gsm_context* c, uint64_t* stream) {
  if (!c || !stream) return set_error(GSM_ERR_VALUE, "null context or output");
  *stream = (uint64_t)(uintptr_t)c->stream;
  return GSM_OK;
}

gsm_status gsm_context_free(gsm_context* c) {
  if (!c) return GSM_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  ctx_clear_graphs(c);
  if (c->arena) cudaFree(c->arena);
  if (c->d_status) cudaFree(c->d_status);
  if (c->d_block) cudaFree(c->d_block);
  if (c->d_ctr) cudaFree(c->d_ctr);
  if (c->d_slice) cudaFree(c->d_slice);
  if (c->h_block) cudaFreeHost(c->h_block);
  if (c->d_slots) cudaFree(c->d_slots);
  if (c->d_chunks) cudaFree(c->d_chunks);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->d_stage) cudaFree(c->d_stage);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->ev_q0) cudaEventDestroy(c->ev_q0);
  if (c->ev_q1) cudaEventDestroy(c->ev_q1);
  if (c->ev_q2) cudaEventDestroy(c->ev_q2);
  for (cudaEvent_t ev : {c->ev_b0, c->ev_b1, c->ev_done, c->ev_fork, c->ev_ext})
    if (ev) cudaEventDestroy(ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return GSM_OK;
}

struct QueryArgs {
  const gsm_pattern* steps;
  int32_t n;
  const int32_t* proj;
  int32_t n_proj;
  int32_t distinct;
  int64_t budget;
  int32_t budget_mode;
  int64_t part, parts;
  gsm_report* rep;
  // Seeded execution (gsm_execute_seeded): step 0 is this device table
  // (row-major seed_n x seed_k) instead of a scan; seed_k < 0 = not seeded.
  const u32* seed = nullptr;
  int64_t seed_n = 0;
  const int32_t* seed_vars = nullptr;
  int32_t seed_k = -1;
};

// Per-query host state between launch and completion.
struct ExecState {
  Exec ex;
  int pack_stat = 0;
  i64 pack_cap = 0;
  u32* pack_out = nullptr;
  bool fused = false;
  int kernels = 0;
  i64 h2d = 0;
  bool allow_fuse = true;
  bool timing = false;
  std::string plan_key;
  std::vector<int> kinds, arities;  // per step (report, budget checks)
  std::vector<int> fused_in;        // per step: 1 = ran inside the previous step's kernel
  // Batch capture: the caller holds c->stream inside a stream capture; only
  // issue the launch sequence into it and describe it in `meta`.
  bool capture_only = false;
  // a one-query timed batch: the context's ev_b0 / ev_b1 are recorded as the
  // first and last nodes of the query's own sequence (device time without
  // the host's graph submission, as for batch graphs)
  bool span_events = false;
  char* pre_image = nullptr;  // batch capture: the d_image buffer to use
  bool zc = false;            // counters and result rows written straight to pinned host memory
  bool big = false;           // this plan's last result outgrew the staging buffer
  gsm_context::GraphEntry meta;
  cudaStream_t sync_stream = nullptr;  // first completion waits here (batch graph)
  bool synced = false;                 // ... or the caller already waited for it
};

// Restore a prepared plan into the context: query-block image with fresh
// epochs, and the host-side facts the completion needs.
// Epochs a replay takes from the device counter: k_init's (install
// variant) plus, for a self-cleaning plan, the next replay's at its end.
static int replay_epochs(const gsm_context::GraphEntry& P, bool warm) {
  return warm ? P.n_epochs : (P.self_clean ? 2 * P.n_epochs : P.n_epochs);
}
static void apply_entry(gsm_context* c, const gsm_context::GraphEntry& P, ExecState& S,
                        bool warm = false) {
  reserve_epochs(c, replay_epochs(P, warm));
  S.zc = P.zc;
  S.pack_stat = P.pack_stat;
  S.pack_cap = P.pack_cap;
  S.pack_out = P.pack_out;
  S.fused = P.fused;
  S.kernels = P.kernels;
  S.h2d = P.h2d;
  S.kinds = P.kinds;
  S.arities = P.arities;
  S.fused_in = P.fused_in;
}

// Plan key: everything a query's launch sequence derives from, including the
// D2H size guess (the last result size of this plan rounded up to a power of
// two, >= 4 KiB, else 64 KiB; never more than the staging buffer), which this
// sets in c->guess.  S.plan_key gets the key without the guess.
static std::string query_key(gsm_context* c, const QueryArgs& qa, ExecState& S) {
  std::string key;
  auto put = [&key](const void* p, size_t b) { key.append(reinterpret_cast<const char*>(p), b); };
  put(qa.steps, sizeof(gsm_pattern) * (size_t)qa.n);
  put(qa.proj, sizeof(int32_t) * (size_t)qa.n_proj);
  const i64 scal[] = {qa.n,     qa.n_proj, qa.distinct != 0, S.allow_fuse, S.timing,
                      qa.budget, qa.part,   qa.parts,         S.span_events};
  put(scal, sizeof scal);
  auto lb = c->last_bytes.find(key);
  size_t g = 65536;
  if (lb != c->last_bytes.end()) {
    g = 4096;
    while (g < lb->second) g <<= 1;
  }
  c->guess = std::min(g, c->stage_bytes);
  S.big = lb != c->last_bytes.end() && lb->second > c->stage_bytes;
  S.plan_key = key;
  key.append(reinterpret_cast<const char*>(&c->guess), sizeof c->guess);
  key.push_back(S.big ? 'B' : 'S');
  key.push_back(c->use_row_hints && c->row_hints.count(S.plan_key) ? 'H' : 'U');  // grids from rows seen
  return key;
}

// Plan the query and enqueue its whole launch sequence (as a CUDA graph
// replay when possible) on the context's stream.  Does not synchronize.
static gsm_status launch_query(gsm_context* c, const QueryArgs& qa, ExecState& S) {
  const gsm_pattern* steps = qa.steps;
  const int32_t n = qa.n;
  const int32_t* proj = qa.proj;
  const int32_t n_proj = qa.n_proj;
  const int64_t budget = qa.budget;
  const int64_t part = qa.part, parts = qa.parts;
  const bool timing = S.timing, distinct = qa.distinct != 0, allow_fuse = S.allow_fuse;
  S.ex = Exec{};
  c->gen++;
  Exec& ex = S.ex;
  int& pack_stat = S.pack_stat;
  i64& pack_cap = S.pack_cap;
  u32*& pack_out = S.pack_out;
  int& kernels = S.kernels;
  i64& h2d = S.h2d;
  kernels = 0;
  QueryBlock* hb = c->h_block;
  cudaStream_t st = c->stream;

  std::string key = query_key(c, qa, S);

  // Prepared plan: replay the captured launch sequence with the saved
  // query-block image and fresh epochs — no re-planning on the host.
  // (Seeded queries read a caller buffer: never cached.)
  // (a left-row chunk of many is run once: not worth a capture)
  const bool graphs = c->use_graphs && qa.seed_k < 0 && !S.capture_only && qa.parts < 64;
  if (graphs) {
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) {
      const gsm_context::GraphEntry& P = it->second;
      const bool warm = P.warm && c->installed == P.image_id;
      apply_entry(c, P, S, warm);
      if (warm) kernels--;  // no k_init
      GSM_CUDA(cudaGraphLaunch(warm ? P.warm : P.exec, st));
      c->installed = P.self_clean ? P.image_id : 0;
      count_launch(kernels);
      return GSM_OK;
    }
  }
  c->installed = 0;  // the block is about to be rewritten by a fresh plan
  ex.c = c;
  ex.steps = steps;
  ex.n = n;
  if (c->use_row_hints) {
    auto rh = c->row_hints.find(S.plan_key);
    if (rh != c->row_hints.end()) ex.hint = &rh->second;
  }
  ex.hb = hb;
  ex.half = c->arena_bytes / 2;
  ex.plan.assign(n, StepPlan());
  memset(hb->stats, 0, sizeof(hb->stats));
  memset(hb->counters, 0, sizeof(hb->counters));
  memset(hb->qcount, 0, sizeof(hb->qcount));
  memset(hb->qhead, 0, sizeof(hb->qhead));
  memset(hb->done, 0, sizeof(hb->done));

  DTable* dT = c->d_block->tables;
  StepStat* dS = c->d_block->stats;
  u32* dC = c->d_block->counters;

  // ---- step 0: scan ----
  int cur;
  std::vector<int> schema;
  if (qa.seed_k >= 0) {  // the caller's table, transposed into arena half A
    cur = ex.new_table(qa.seed_k, H_A);
    hb->tables[cur].n = qa.seed_n;
    ex.ub[cur] = qa.seed_n;
    hb->stats[0].rows = qa.seed_n;
    schema.assign(qa.seed_vars, qa.seed_vars + qa.seed_k);
  } else {
    cur = ex.scan_table(steps[0], 0);
    schema = pattern_schema(steps[0]);
  }
  ex.plan[0].kind = S_SCAN;
  ex.plan[0].schema = schema;
  ex.plan[0].out_table = cur;

  // ---- plan the joins (executor.py:340-356) and build right tables ----
  struct Launch {
    StepKind kind;
    int step, left, right, out;
    ExpandP ep;
    FilterP fp;
    GroupP gp;
    int a, b;
    int grid;
    int last_step;  // S_GROUP: the last fused step
    u32 fanout;     // S_EXPAND: longest candidate run of the orientation
    bool drain;     // hub pieces may be queued: launch k_drain after
    int items;      // S_EXPAND: rows per thread of a tile (1 or 2)
    i64 avg_run;    // S_EXPAND / S_GROUP: average candidate run of the expanded orientation
  };
  std::vector<Launch> launches;
  // Step fusion state: a group is [filters][expand][filters] over one input
  // table; every fused step writes (if at all) to the buffer opposite the
  // group's input, so the group's final table never aliases its input.
  bool g_open = false, g_has_x = false;
  int g_npre = 0, g_npost = 0;
  u32 g_x_fanout = 0;  // longest candidate list of the group's expand
  i64 g_x_avg = 0, g_x_est = 0;  // its average run, expected output rows
  Home g_in_home = H_NONE;
  int g_x_var = -1;    // the variable the group's expand binds
  int g_x_step = -1;   // ... and its plan step
  // Candidates per left row of the group's expand: the orientation's
  // average run, or — once the plan has run (row hints) — what the expand
  // actually produced per left row (LUBM-1000 c3: average run >= 4 but 0.15
  // candidates per left row, since most left keys have no run at all)
  auto x_yield = [&]() -> i64 {
    if (ex.hint && g_x_step >= 1 && g_x_step < (int)ex.hint->size()) {
      const i64 l = (*ex.hint)[g_x_step - 1], o = (*ex.hint)[g_x_step];
      return l > 0 ? o / l : 0;
    }
    return g_x_avg;
  };
  std::vector<int> group_id(n, -1);
  int n_groups = 0;
  Orient slice_R{};  // the first join's orientation / left key column: equal-E partition
  int slice_key = -1;
  for (int s = 1; s < n; s++) {
    const gsm_pattern& p = steps[s];
    std::vector<int> rs = pattern_schema(p);
    std::vector<int> jv;
    for (int v : schema)
      if (index_of(rs, v) >= 0) jv.push_back(v);
    const PredDev* m = ex.pred(p);
    Launch L{};
    L.step = s;
    L.left = cur;
    std::vector<int> out_schema = schema;
    if (jv.empty()) {
      for (int v : rs) out_schema.push_back(v);
    } else {
      for (int v : rs)
        if (index_of(schema, v) < 0) out_schema.push_back(v);
    }
    if ((int)out_schema.size() > GSM_MAX_VARS)
      return set_error(GSM_ERR_VALUE, "query binds more than " + std::to_string(GSM_MAX_VARS) + " variables");
    const int a = (int)schema.size();
    if (!m || jv.empty()) g_open = false;  // empty / cross / gate steps end a fusion group
    if (!m) {
      // R6 right side: the join (or cross product) is empty, E = 0.
      L.kind = S_EMPTY;
      L.out = ex.new_table((int)out_schema.size(), H_NONE);
    } else if (jv.empty()) {
      int rt = ex.scan_table(p, -1);
      L.right = rt;
      if (rs.empty()) {
        L.kind = S_GATE;
        L.out = ex.new_table(a, ex.home[cur]);
      } else {
        L.kind = S_CROSS;
        L.out = ex.new_table((int)out_schema.size(), Exec::other(ex.home[cur]));
        L.a = a;
        L.b = (int)rs.size();
      }
    } else {
      bool sv = p.s_var >= 0, ov = p.o_var >= 0;
      const bool is_expand = sv && ov && p.s_var != p.o_var && jv.size() == 1;
      // join the open group when the [F*][E][F*] shape allows it
      // Filters after the expand run per candidate inside the row's thread,
      // so they are fused only when every candidate list is short (a large
      // fan-out is better spread over blocks by materialising the expand).
      bool join = false;
      if (c->use_fusion && g_open) {
        if (is_expand) join = !g_has_x;
        else if (g_has_x)  // short runs, or an intermediate too large to materialise well,
                           // or a filter whose key is bound before the expand: a sorted-run
                           // intersection per row (its segment looked up once per row)
          join = g_npost < MAXF && (g_x_fanout <= FUSE_MAX_FANOUT ||
                                    (g_x_est >= c->fuse_huge && g_x_fanout <= 64 * std::max<i64>(1, g_x_avg)) ||
                                    (c->use_intersect && g_npost < HOIST && jv[0] != g_x_var &&
                                     g_x_fanout < INTERSECT_MAX_FANOUT && x_yield() >= INTERSECT_MIN_AVG));
        else join = g_npre < MAXF;
      }
      if (!join) {
        g_open = true;
        g_has_x = false;
        g_npre = g_npost = 0;
        g_in_home = ex.home[cur];
        n_groups++;
      }
      if (is_expand) {
        g_has_x = true;
        g_x_step = s;
        g_x_var = jv[0] == p.s_var ? p.o_var : p.s_var;
        const bool on_s = jv[0] == p.s_var;
        const HostAux& gha = on_s ? c->store->aux_so[p.pid] : c->store->aux_os[p.pid];
        g_x_fanout = gha.max_run;
        // expected expand output: left rows x the orientation's average run
        g_x_avg = gha.key.empty() ? 0 : (i64)(gha.off.back() / gha.key.size());
        g_x_est = Exec::sat_mul(ex.ub[cur], std::max<i64>(1, g_x_avg));
      } else if (g_has_x) g_npost++;
      else g_npre++;
      group_id[s] = n_groups - 1;
      const Home oh = Exec::other(g_in_home);
      if (is_expand) {
        L.kind = S_EXPAND;
        L.out = ex.new_table((int)out_schema.size(), oh);
        ExpandP& e = L.ep;
        bool on_s = jv[0] == p.s_var;
        e.R = on_s ? m->so : m->os;
        e.li = index_of(schema, jv[0]);
        e.a = a;
        e.L = dT + cur;
        e.out = reinterpret_cast<u32*>(ex.buf(oh));
        e.cap = ex.cap_for((int)out_schema.size());
        e.O = dT + L.out;
        e.st = dS + s;
        L.fanout = (on_s ? c->store->aux_so[p.pid] : c->store->aux_os[p.pid]).max_run;
        if (s == 1) {
          slice_R = e.R;
          slice_key = e.li;
        }
      } else {
        L.kind = S_FILTER;
        L.out = ex.new_table(a, oh);
        FilterP& f = L.fp;
        f.a = a;
        f.L = dT + cur;
        f.out = reinterpret_cast<u32*>(ex.buf(oh));
        f.cap = ex.cap_for(a);
        f.O = dT + L.out;
        f.st = dS + s;
        f.li = index_of(schema, jv[0]);
        f.lj = -1;
        f.cval = 0;
        if (sv && ov && p.s_var != p.o_var) {  // J2: first join var drives (executor.py:141-145)
          f.mode = F_PAIR;
          bool on_s = jv[0] == p.s_var;
          f.R = on_s ? m->so : m->os;
          f.lj = index_of(schema, on_s ? p.o_var : p.s_var);
          if (s == 1) {
            slice_R = f.R;
            slice_key = f.li;
          }
        } else if (sv && ov) {  // R4 (?x p ?x)
          f.mode = F_SELF;
          f.R = m->so;
        } else if (sv) {  // R2 (?s p C): (s, C) in M
          f.mode = F_CONST;
          f.R = m->so;
          f.cval = p.o_const;
        } else {  // R3 (C p ?o): (C, o) in M
          f.mode = F_CONST;
          f.R = m->os;
          f.cval = p.s_const;
        }
      }
    }
    // host-side row bounds -> grid sizes (any grid is correct: blocks are persistent)
    const i64 lub = ex.ub[cur];
    switch (L.kind) {
      case S_EMPTY: ex.ub[L.out] = 0; break;
      case S_FILTER: ex.ub[L.out] = lub; break;
      case S_GATE: ex.ub[L.out] = lub; break;
      case S_CROSS: ex.ub[L.out] = Exec::sat_mul(lub, ex.ub[L.right]); break;
      case S_EXPAND: {
        const bool on_s = jv[0] == p.s_var;
        const HostAux& ha = on_s ? c->store->aux_so[p.pid] : c->store->aux_os[p.pid];
        ex.ub[L.out] = Exec::sat_mul(lub, (i64)ha.max_run);
        break;
      }
      default: break;
    }
    // Large left tables over short runs: 512-row tiles (two rows per thread)
    // halve the number of tiles a block walks through one after another,
    // each paying its count -> scan -> look-back latency once (power-law 100M:
    // chain2 0.73 -> 0.56 ms, chain3 0.54 -> 0.37 ms).  Not for few tiles
    // (fewer blocks busy) or long runs (the tile's own work dominates).
    L.items = 1;
    L.avg_run = 0;
    if (L.kind == S_EXPAND) {
      const bool on_s = jv[0] == p.s_var;
      const HostAux& ha = on_s ? c->store->aux_so[p.pid] : c->store->aux_os[p.pid];
      const i64 avg_run = ha.key.empty() ? 0 : (i64)(ha.off.back() / ha.key.size());
      L.avg_run = avg_run;
      L.items = c->tile_items > 0 ? c->tile_items
                                  : (lub >= (i64)16 * c->grid_ts * TS_TILE && avg_run <= 16 ? 2 : 1);
      // 512-row tiles stage at most 4 left columns for their window scatter
    }
    L.grid = L.kind == S_CROSS ? ex.grid_for_rows(ex.hinted(L.out, s), 256)
                               : ex.grid_for_rows(ex.hinted(cur, s - 1), TS_TILE * L.items);
    ex.plan[s].kind = L.kind;
    ex.plan[s].schema = out_schema;
    ex.plan[s].out_table = L.out;
    launches.push_back(L);
    schema = out_schema;
    cur = L.out;
  }

  // ---- fuse each multi-step group into one k_group launch ----
  if (c->use_fusion) {
    std::vector<Launch> fl;
    size_t i = 0;
    while (i < launches.size()) {
      const int gid = group_id[launches[i].step];
      size_t j = i + 1;
      if (gid >= 0)
        while (j < launches.size() && group_id[launches[j].step] == gid) j++;
      if (gid < 0 || j - i == 1) {
        fl.push_back(launches[i]);
        i = j;
        continue;
      }
      Launch G{};
      G.kind = S_GROUP;
      G.step = launches[i].step;
      G.last_step = launches[j - 1].step;
      G.left = launches[i].left;
      G.out = launches[j - 1].out;
      G.grid = launches[i].grid;
      GroupP& gp = G.gp;
      gp.L = dT + G.left;
      gp.a = ex.arity[G.left];
      std::vector<FSpec> pre, post;
      for (size_t k = i; k < j; k++) {
        const Launch& L = launches[k];
        const int slot = gp.nslots++;
        gp.st[slot] = dS + L.step;
        if (L.kind == S_EXPAND) {
          gp.has_x = 1;
          gp.X = L.ep.R;
          gp.xk = L.ep.li;
          gp.xslot = slot;
          G.fanout = L.fanout;
          G.avg_run = L.avg_run;
          G.items = 1;
        } else {
          FSpec fs{L.fp.R, L.fp.mode, L.fp.li, L.fp.lj, L.fp.cval, slot};
          (gp.has_x ? post : pre).push_back(fs);
        }
      }
      gp.npre = (int)pre.size();
      gp.npost = (int)post.size();
      for (int q = 0; q < gp.npre; q++) gp.f[q] = pre[q];
      for (int q = 0; q < gp.npost; q++) gp.f[gp.npre + q] = post[q];
      gp.last_slot = gp.nslots - 1;
      const Launch& last = launches[j - 1];
      gp.out = last.kind == S_EXPAND ? last.ep.out : last.fp.out;
      gp.cap = last.kind == S_EXPAND ? last.ep.cap : last.fp.cap;
      gp.O = dT + G.out;
      fl.push_back(G);
      i = j;
    }
    launches.swap(fl);
  }
  S.fused_in.assign(n, 0);
  for (const Launch& L : launches)
    if (L.kind == S_GROUP)
      for (int q = L.step + 1; q <= L.last_step; q++) S.fused_in[q] = 1;

  // ---- hub deferral for expands whose orientation has long runs ----
  {
    int slot = 0;
    for (auto& L : launches) {
      if (L.kind != S_EXPAND && L.kind != S_FILTER && L.kind != S_GROUP) continue;
      // Rows of >= DEFER_ROW candidates when the left table is small (few
      // tiles: the hubs would serialise on a few blocks); with many tiles the
      // blocks already share rows of that size, and only true hubs
      // (>= DEFER_BIG) are worth the queue round trip.
      const bool small_left = ex.ub[L.left] <= (i64)c->grid_ts * TS_TILE / 4;
      const u32 min_len = small_left ? (u32)DEFER_ROW : (u32)DEFER_BIG;
      const i64 heavy = std::max<i64>(HEAVY_TILE, 16 * L.avg_run * (i64)TS_TILE * std::max(1, L.items));
      const bool hubby = c->use_defer && L.fanout >= (u32)DEFER_ROW;
      if (hubby && L.kind == S_EXPAND) {
        L.ep.dq = ChunkQueue{c->d_chunks, c->d_block->qcount + slot, c->d_block->qhead + slot,
                             c->chunk_cap, min_len, heavy};
        L.drain = true;
      } else if (hubby && L.kind == S_GROUP && L.gp.has_x && L.gp.npost == 0) {
        L.gp.dq = ChunkQueue{c->d_chunks, c->d_block->qcount + slot, c->d_block->qhead + slot,
                             c->chunk_cap, min_len, heavy};
        L.drain = true;
      }
      slot++;
    }
  }

  // ---- projection target ----
  int pj_idx[GSM_MAX_VARS];
  if (n_proj > GSM_MAX_VARS) return set_error(GSM_ERR_VALUE, "too many projected variables");
  for (int j = 0; j < n_proj; j++) {
    pj_idx[j] = index_of(schema, proj[j]);
    if (pj_idx[j] < 0) return set_error(GSM_ERR_VALUE, "projected variable is not bound by the plan");
  }
  Home ph = ex.home[cur] == H_A ? H_B : H_A;
  pack_out = reinterpret_cast<u32*>(ex.buf(ph));
  pack_cap = n_proj ? (i64)(ex.half / (4 * (size_t)n_proj)) : ((i64)1 << 62);
  pack_stat = n;
  // Zero-copy results: when this plan's last result was small, the last
  // kernel writes the step counters and the projected rows straight into the
  // pinned staging buffer (no device->host copy in the launch sequence).
  // Results packed by k_pack (plans ending in a scan) are written row after
  // row with coalesced stores, so they stay zero-copy up to ZC_PACK_BYTES;
  // the joins' fused projections scatter, so their limit is ZC_BYTES.
  const bool packs = launches.empty() && !distinct && qa.seed_k < 0 && n_proj >= 1 && n_proj <= 2;
  const size_t zc_lim = packs ? ZC_PACK_BYTES : c->zc_bytes;
  S.zc = c->guess <= zc_lim;
  const size_t stage_lim = S.zc ? std::min<size_t>(c->stage_bytes, zc_lim) : c->stage_bytes;
  const i64 stage_cap = n_proj ? (i64)(stage_lim / (4 * (size_t)n_proj)) : ((i64)1 << 62);
  u32* const stage_rows = S.zc ? c->hd_rows : c->d_rows;
  // Fuse the projection into the last join when it is an expand/filter and
  // the result goes to the host staging buffer (no DISTINCT).
  // Results that outgrew the staging buffer last time (S.big) are written
  // by the last join into its own (otherwise unused) arena half instead: a
  // device-resident result without the k_pack pass.
  bool fused = false;
  const Home big_home = launches.empty() ? H_NONE : ex.home[launches.back().out];
  if (allow_fuse && c->use_proj_fusion && !distinct && !launches.empty() && n_proj > 0 &&
      (launches.back().kind == S_EXPAND || launches.back().kind == S_FILTER ||
       launches.back().kind == S_GROUP) &&
      (!S.big || big_home == H_A || big_home == H_B)) {
    FusedOut fz;
    if (S.big) {
      fz.stage = reinterpret_cast<u32*>(ex.buf(big_home));
      fz.cap = (i64)(ex.half / (4 * (size_t)n_proj));
      fz.dev = 1;
      pack_out = fz.stage;
      pack_cap = fz.cap;
    } else {
      fz.stage = stage_rows;
      fz.cap = stage_cap;
    }
    fz.k = n_proj;
    for (int j = 0; j < n_proj; j++) fz.pj[j] = pj_idx[j];
    fz.pst = dS + pack_stat;
    if (launches.back().kind == S_EXPAND) launches.back().ep.fz = fz;
    else if (launches.back().kind == S_FILTER) launches.back().fp.fz = fz;
    else launches.back().gp.fz = fz;
    fused = true;
  }
  S.fused = fused;

  // ---- per-launch epochs: data in the query block, so a captured graph
  //      replays with fresh epochs and unchanged kernel parameters ----
  int n_epoch_slots = 0;
  for (auto& L : launches)
    if (L.kind == S_EXPAND || L.kind == S_FILTER || L.kind == S_GROUP)
      n_epoch_slots++;
  // k_init takes them from the device counter; mirror it (any wrap-around
  // re-zeroing is enqueued here, before a capture starts — a batch capture
  // made room beforehand, epoch_headroom).  A self-cleaning plan's last
  // kernel takes the next replay's epochs as well.
  const bool self_clean = c->use_self_clean && (graphs || S.capture_only) && !distinct && qa.seed_k < 0;
  reserve_epochs(c, self_clean ? 2 * n_epoch_slots : n_epoch_slots);
  ProjArgs pa{};
  for (int j = 0; j < n_proj; j++) pa.col[j] = pj_idx[j];
  const size_t used = offsetof(QueryBlock, tables) + sizeof(DTable) * (size_t)ex.ntables;
  h2d = (i64)used;

  // The whole query as one stream-ordered sequence: H2D of the query block,
  // the kernels, D2H of the step counters.  Nothing here writes host memory.
  bool capturing = false;
  // Graph modes: the device image of the query block that k_init copies.
  char* d_image = nullptr;
  if (S.capture_only) {
    d_image = S.pre_image;
  } else if (graphs) {
    GSM_CUDA(cudaMalloc(&d_image, sizeof(QueryBlock)));
    // k_init copies whole 16-byte words: the tail past `used` must be defined
    cudaError_t ce = cudaMemset(d_image, 0, sizeof(QueryBlock));
    if (ce == cudaSuccess) ce = cudaMemcpy(d_image, hb, used, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
      cudaFree(d_image);
      return cuda_error(ce, "cudaMemcpy(query image)");
    }
  }
  // Under stream capture an event record must be an external node to be
  // timeable; outside capture the flag is illegal.
  auto record = [&](cudaEvent_t ev) -> cudaError_t {
    return capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                     : cudaEventRecord(ev, st);
  };
  // warm: the self-cleaning variant without k_init (the block already holds
  // this plan's image, left clean by its previous replay)
  auto issue = [&](bool warm) -> gsm_status {
    int nk = 0;
    if (S.span_events) GSM_CUDA(record(c->ev_b0));
    if (timing) GSM_CUDA(record(c->ev_q0));
    // the query block: a replayed graph copies its device image in k_init;
    // otherwise it is uploaded here
    if (!d_image) GSM_CUDA(cudaMemcpyAsync(c->d_block, hb, used, cudaMemcpyHostToDevice, st));
    if (timing) GSM_CUDA(record(c->ev[0]));  // step 0 (scan) = k_init's constant resolution
    if (!warm) {
      QueryBlock* img = reinterpret_cast<QueryBlock*>(d_image);
      GSM_CUDA(launch(c->use_pdl, k_init, 1, 256, st, reinterpret_cast<const uint4*>(d_image),
                      reinterpret_cast<uint4*>(c->d_block), d_image ? (int)((used + 15) / 16) : 0, c->d_ctr,
                      c->d_block->epochs, n_epoch_slots, ex.res, dT, dS,
                      img ? img->tables : nullptr, img ? img->stats : nullptr));
      nk++;
    }
    if (qa.seed_k > 0 && qa.seed_n > 0) {
      const i64 cells = qa.seed_n * qa.seed_k;
      k_rows_to_cols<<<(int)std::max<i64>(1, std::min<i64>(c->grid_ts, (cells + 255) / 256)), 256, 0, st>>>(
          qa.seed, qa.seed_n, qa.seed_k, reinterpret_cast<u32*>(ex.buf(H_A)), ex.cap_for(qa.seed_k));
      GSM_CUDA(cudaGetLastError());
      nk++;
    }
    if (parts > 1 && slice_key >= 0 && c->d_slice && c->use_equal_e) {
      const i64 nch = std::min<i64>(ex.ub[ex.plan[0].out_table], SLICE_CHUNKS);
      GSM_CUDA(launch(c->use_pdl, k_slice_sums, (int)std::max<i64>(1, std::min<i64>(c->grid_ts, (nch + 7) / 8)),
                      256, st, (const DTable*)(dT + ex.plan[0].out_table), slice_key, slice_R, c->d_slice));
      GSM_CUDA(launch(c->use_pdl, k_slice_pick, 1, 1024, st, dT + ex.plan[0].out_table,
                      (int)ex.plan[0].schema.size(), part, parts, dS + 0, (const u64*)c->d_slice,
                      slice_key, slice_R));
      nk += 2;
    } else if (parts > 1) {
      GSM_CUDA(launch(c->use_pdl, k_slice, 1, 64, st, dT + ex.plan[0].out_table,
                      (int)ex.plan[0].schema.size(), part, parts, dS + 0));
      nk++;
    }
    if (timing) GSM_CUDA(record(c->ev[1]));
    // the query's last kernel exports the step counters to the stage head
    // (and, self-cleaning, restores the block for the next replay)
    ExportArgs xlast{dS, reinterpret_cast<StepStat*>(S.zc ? c->hd_stage : c->d_stage), n + 1,
                     c->d_block->done};
    if (self_clean) {
      xlast.img = reinterpret_cast<const uint4*>(d_image);
      xlast.blk = reinterpret_cast<uint4*>(c->d_block);
      xlast.words16 = (int)((used + 15) / 16);
      xlast.ctr = c->d_ctr;
      xlast.epochs = c->d_block->epochs;
      xlast.n_epochs = n_epoch_slots;
    }
    int last_launch = -1;
    for (int i = (int)launches.size() - 1; i >= 0 && fused; i--)
      if (launches[i].kind != S_EMPTY) {
        last_launch = i;
        break;
      }
    int slot = 0;
    for (int li = 0; li < (int)launches.size(); li++) {
      auto& L = launches[li];
      const bool is_last = li == last_launch;
      const ExportArgs xm = is_last && !L.drain ? xlast : ExportArgs{};
      const ExportArgs xd = is_last && L.drain ? xlast : ExportArgs{};
      switch (L.kind) {
        case S_EMPTY:
          break;  // descriptor n = 0 and zero stats were uploaded
        case S_EXPAND: {
          TileSync ts{c->d_status, dC + slot, c->d_block->epochs + slot, 0};
          slot++;
          if (L.items == 2)
          {
            // count-ahead 512-row tiles stage 4 left columns; wider tables
            // take the one-buffer variant (8 columns, static shared memory)
            if (L.ep.a <= ExpandP::win_a<2 * TS_THREADS, 2>())
              GSM_CUDA(launch_smem(c->use_pdl, ExpandP::lt_bytes<2 * TS_THREADS, 2>(),
                                   k_tilescan<ExpandP, 2, true>, L.grid, TS_THREADS, st, L.ep, ts, xm));
            else
              GSM_CUDA(launch(c->use_pdl, k_tilescan<ExpandP, 2, false>, L.grid, TS_THREADS, st, L.ep,
                              ts, xm));
          }
          else
            GSM_CUDA(launch(c->use_pdl, k_tilescan<ExpandP>, L.grid, TS_THREADS, st, L.ep, ts, xm));
          nk++;
          if (L.drain) {
            GSM_CUDA(launch(c->use_pdl, k_drain<ExpandP>, c->grid_ts, TS_THREADS, st, L.ep, L.ep.dq, xd));
            nk++;
          }
          break;
        }
        case S_FILTER: {
          TileSync ts{c->d_status, dC + slot, c->d_block->epochs + slot, 0};
          slot++;
          GSM_CUDA(launch(c->use_pdl, k_tilescan<FilterP>, L.grid, TS_THREADS, st, L.fp, ts, xm));
          nk++;
          break;
        }
        case S_GROUP: {
          TileSync ts{c->d_status, dC + slot, c->d_block->epochs + slot, 0};
          slot++;
          GSM_CUDA(launch(c->use_pdl, k_group, L.grid, TS_THREADS, st, L.gp, ts, xm));
          nk++;
          if (L.drain) {
            GSM_CUDA(launch(c->use_pdl, k_drain<GroupEmit>, c->grid_ts, TS_THREADS, st,
                            GroupEmit{L.gp}, L.gp.dq, xd));
            nk++;
          }
          break;
        }
        case S_CROSS: {
          Home oh = ex.home[L.out];
          GSM_CUDA(launch(c->use_pdl, k_cross, L.grid, 256, st, (const DTable*)(dT + L.left),
                          (const DTable*)(dT + L.right), L.a, L.b,
                          reinterpret_cast<u32*>(ex.buf(oh)), ex.cap_for(L.a + L.b), (i64)budget,
                          dT + L.out, dS + L.step, ExportArgs{}));
          nk++;
          break;
        }
        case S_GATE:
          GSM_CUDA(launch(c->use_pdl, k_gate, 1, 64, st, (const DTable*)(dT + L.left),
                          (const DTable*)(dT + L.right), ex.arity[L.left], dT + L.out, dS + L.step,
                          ExportArgs{}));
          nk++;
          break;
        default:
          break;
      }
      if (timing) {
        const int last = L.kind == S_GROUP ? L.last_step : L.step;
        for (int q = L.step; q <= last; q++)  // fused steps: the group's time is on its first step
          GSM_CUDA(record(c->ev[q + 1]));
      }
    }
    if (!fused) {
      // DISTINCT reads the packed rows on the device, so only plain
      // projections are packed straight into the pinned staging buffer.
      u32* host_dst = distinct ? nullptr : stage_rows;
      GSM_CUDA(launch(c->use_pdl, k_pack, ex.grid_for_rows(ex.hinted(cur, n - 1), 256), 256, st,
                      (const DTable*)(dT + cur), pa, n_proj, pack_out, pack_cap, host_dst,
                      stage_cap, dS + pack_stat, xlast));
      nk++;
    }
    if (timing) GSM_CUDA(record(c->ev_q1));
    GSM_CUDA(cudaGetLastError());
    // Not zero-copy: ONE copy of the step counters (exported by the last
    // kernel) and the result rows up to this plan's expected size; the host
    // fetches any remainder after the sync (rare: only when the result grew).
    if (!S.zc)
      GSM_CUDA(cudaMemcpyAsync(c->h_stage, c->d_stage, STAGE_HEAD + ((distinct || S.big) ? 0 : c->guess),
                               cudaMemcpyDeviceToHost, st));
    if (S.span_events) GSM_CUDA(record(c->ev_b1));
    kernels = nk;
    return GSM_OK;
  };

  S.kinds.resize(n);
  S.arities.resize(n);
  for (int q = 0; q < n; q++) {
    S.kinds[q] = (int)ex.plan[q].kind;
    S.arities[q] = (int)ex.plan[q].schema.size();
  }
  if (S.capture_only) {  // the caller's capture records the sequence
    capturing = true;
    gsm_status is = issue(false);  // with k_init: the batch toggles its node per launch
    capturing = false;
    if (is != GSM_OK) return is;
    gsm_context::GraphEntry& P = S.meta;
    P.kernels = kernels;
    P.self_clean = self_clean;
    P.image.assign(reinterpret_cast<const char*>(hb), reinterpret_cast<const char*>(hb) + used);
    P.n_epochs = n_epoch_slots;
    P.pack_stat = pack_stat;
    P.pack_cap = pack_cap;
    P.pack_out = pack_out;
    P.fused = S.fused;
    P.h2d = h2d;
    P.zc = S.zc;
    P.d_image = d_image;
    P.kinds = S.kinds;
    P.arities = S.arities;
    P.fused_in = S.fused_in;
    return GSM_OK;
  }
  if (graphs) {
    cudaGraphExec_t ge = nullptr;
    {
      if (c->graphs.size() >= 1024) ctx_clear_graphs(c);
      // the install variant (k_init first) and, self-cleaning, the warm one
      cudaGraphExec_t gw = nullptr;
      int nk_install = 0;
      for (int v = 0; v < (self_clean ? 2 : 1); v++) {
        GSM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        gsm_status is = issue(v == 1);
        capturing = false;
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &g);
        cudaGraphExec_t* dst = v == 0 ? &ge : &gw;
        if (is == GSM_OK && ce == cudaSuccess) ce = cudaGraphInstantiate(dst, g, 0);
        if (g) cudaGraphDestroy(g);
        if (is != GSM_OK || ce != cudaSuccess) {
          if (ge) cudaGraphExecDestroy(ge);
          cudaFree(d_image);
          return is != GSM_OK ? is : cuda_error(ce, "graph capture");
        }
        if (v == 0) nk_install = kernels;
      }
      kernels = nk_install;
      gsm_context::GraphEntry P;
      P.exec = ge;
      P.warm = gw;
      P.self_clean = self_clean;
      P.image_id = next_image_id();
      P.kernels = kernels;
      P.image.assign(reinterpret_cast<const char*>(hb), reinterpret_cast<const char*>(hb) + used);
      P.n_epochs = n_epoch_slots;
      P.pack_stat = pack_stat;
      P.pack_cap = pack_cap;
      P.pack_out = pack_out;
      P.fused = S.fused;
      P.h2d = h2d;
      P.zc = S.zc;
      P.d_image = d_image;
      P.kinds = S.kinds;
      P.arities = S.arities;
      P.fused_in = S.fused_in;
      c->installed = 0;
      const u64 id = P.image_id;
      c->graphs.emplace(key, std::move(P));
      GSM_CUDA(cudaGraphLaunch(ge, st));
      c->installed = self_clean ? id : 0;
    }
  } else {
    gsm_status is = issue(false);
    if (is != GSM_OK) return is;
  }
  count_launch(kernels);
  return GSM_OK;
}

static gsm_status validate_query(const gsm_context* c, const QueryArgs& q) {
  if (!c) return set_error(GSM_ERR_VALUE, "null context");
  if (q.n <= 0) return set_error(GSM_ERR_VALUE, "cannot execute an empty plan");
  if (q.n > GSM_MAX_STEPS) return set_error(GSM_ERR_VALUE, "plan has more than 64 steps");
  if (!q.steps) return set_error(GSM_ERR_VALUE, "null plan");
  if (q.n_proj < 0 || (q.n_proj > 0 && !q.proj)) return set_error(GSM_ERR_VALUE, "bad projection");
  if (q.parts < 1 || q.part < 0 || q.part >= q.parts) return set_error(GSM_ERR_VALUE, "bad partition");
  if (q.budget_mode != GSM_BUDGET_SEQUENTIAL && q.budget_mode != GSM_BUDGET_PARALLEL)
    return set_error(GSM_ERR_VALUE, "bad budget mode");
  for (int s = 0; s < q.n; s++) {
    const gsm_pattern& p = q.steps[s];
    if (p.s_var >= GSM_MAX_VARS || p.o_var >= GSM_MAX_VARS || p.s_var < -1 || p.o_var < -1)
      return set_error(GSM_ERR_VALUE, "variable index out of range");
  }
  if (q.seed_k >= 0) {
    if (q.seed_k > GSM_MAX_VARS || q.seed_n < 0 || (q.seed_k > 0 && !q.seed_vars) ||
        (q.seed_k > 0 && q.seed_n > 0 && !q.seed))
      return set_error(GSM_ERR_VALUE, "bad seed table");
    for (int i = 0; i < q.seed_k; i++) {
      if (q.seed_vars[i] < 0 || q.seed_vars[i] >= GSM_MAX_VARS)
        return set_error(GSM_ERR_VALUE, "seed variable index out of range");
      for (int j = 0; j < i; j++)
        if (q.seed_vars[j] == q.seed_vars[i]) return set_error(GSM_ERR_VALUE, "duplicate seed variable");
    }
  }
  return GSM_OK;
}

static gsm_status begin_query(gsm_context* c, const QueryArgs& q, ExecState& S) {
  gsm_status v = validate_query(c, q);
  if (v != GSM_OK) return v;
  GSM_CUDA(cudaSetDevice(c->device));
  if (q.seed_k > 0 && q.seed_n > 0) {  // the seed must fit one arena half
    const size_t need = 8 * (size_t)q.seed_k * (size_t)q.seed_n;
    if (c->arena_bytes < need) {
      gsm_status s2 = ctx_set_arena(c, need + need / 4);
      if (s2 != GSM_OK) return s2;
    }
  }
  S.timing = q.rep && q.rep->device_ms;
  return launch_query(c, q, S);
}

// Wait for a launched query, apply the budget rules, re-run on arena /
// staging overflow, and hand the result over.
static gsm_status complete_query(gsm_context* c, const QueryArgs& qa, ExecState& S,
                                 gsm_result** out) {
  *out = nullptr;
  const int32_t n = qa.n, n_proj = qa.n_proj, budget_mode = qa.budget_mode;
  const int64_t budget = qa.budget;
  const bool distinct = qa.distinct != 0, timing = S.timing;
  gsm_report* rep = qa.rep;
  int& pack_stat = S.pack_stat;
  i64& pack_cap = S.pack_cap;
  u32*& pack_out = S.pack_out;
  int& kernels = S.kernels;
  i64& h2d = S.h2d;
  std::string& plan_key = S.plan_key;
  bool tail_event = false;  // DISTINCT ran after the captured sequence
  for (int attempt = 0;; attempt++) {
    if (attempt > 0) {
      gsm_status stt = launch_query(c, qa, S);
      if (stt != GSM_OK) return stt;
    }
    if (!(attempt == 0 && S.synced))
      GSM_CUDA(cudaStreamSynchronize(attempt == 0 && S.sync_stream ? S.sync_stream : c->stream));
    memcpy(c->h_block->stats, c->h_stage, sizeof(StepStat) * (size_t)(n + 1));
    const QueryBlock* hb = c->h_block;
    // Budget checks in plan order (executor.py:158-163, 192-193, 237-241).
    // A step's counters are exact as long as no earlier step overflowed.
    i64 need_rows = 0;
    int need_arity = 1;
    bool ovf = false;
    for (int s = 1; s < n && !ovf; s++) {
      const StepStat& q = hb->stats[s];
      StepKind k = (StepKind)S.kinds[s];
      char msg[256];
      if (k == S_CROSS || k == S_GATE) {
        i64 nl = q.e, nr = q.pad, tot = 0;
        bool big = __builtin_mul_overflow(nl, nr, &tot);
        if (big || tot > budget) {
          snprintf(msg, sizeof msg, "cross product of %lld x %lld rows exceeds budget %lld",
                   (long long)nl, (long long)nr, (long long)budget);
          return set_error(GSM_ERR_RESOURCE, msg);
        }
      } else if (k == S_EXPAND || k == S_FILTER) {
        if (budget_mode == GSM_BUDGET_PARALLEL && q.e > budget) {
          snprintf(msg, sizeof msg, "pre-allocated join region of %lld rows exceeds budget %lld",
                   (long long)q.e, (long long)budget);
          return set_error(GSM_ERR_RESOURCE, msg);
        }
        if (budget_mode == GSM_BUDGET_SEQUENTIAL && q.rows > budget) {
          snprintf(msg, sizeof msg, "join output exceeds row budget %lld", (long long)budget);
          return set_error(GSM_ERR_RESOURCE, msg);
        }
      }
      if (q.overflow) {
        ovf = true;
        need_rows = q.rows;
        need_arity = S.arities[s];
      }
    }
    if (!ovf && hb->stats[pack_stat].overflow) {
      ovf = true;
      need_rows = hb->stats[pack_stat].rows;
      need_arity = n_proj;
    }
    if (!ovf && hb->stats[pack_stat].pad == 3) {
      // The fused projection outgrew the pinned staging buffer (or the
      // zero-copy limit): re-run with a device-side pack, and grow staging
      // (<= 1 GiB) for the next query.
      size_t want = (size_t)hb->stats[pack_stat].rows * 4 * (size_t)std::max(n_proj, 1);
      c->last_bytes[plan_key] = want;
      if (want > c->stage_bytes && want <= c->stage_max) ctx_set_stage(c, want + want / 4);
      S.allow_fuse = false;
      continue;
    }
    if (!ovf) break;
    // Intermediate table larger than the arena half: grow and re-run.
    size_t need = (size_t)need_rows * 4 * (size_t)std::max(need_arity, 1) * 2;
    size_t grow = std::max(need + need / 4, c->arena_bytes * 2);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    size_t avail = free_b + c->arena_bytes;
    if (c->arena_max != ~(size_t)0) avail = std::min(avail, c->arena_max / 9 * 10);
    char msg[256];
    snprintf(msg, sizeof msg, "intermediate result of %lld rows x %d columns exceeds device memory",
             (long long)need_rows, need_arity);
    // GSM_ERR_DEVICE_MEMORY: the host re-runs the plan in left-row chunks
    if (attempt >= 8 || need > (avail * 9) / 10) return set_error(GSM_ERR_DEVICE_MEMORY, msg);
    grow = std::min(grow, (avail * 9) / 10);
    const size_t prev = c->arena_bytes;
    if (ctx_set_arena(c, grow) != GSM_OK) {  // fragmentation: keep the old arena
      cudaGetLastError();
      gsm_status s3 = ctx_set_arena(c, prev);
      if (s3 != GSM_OK) return s3;
      return set_error(GSM_ERR_DEVICE_MEMORY, msg);
    }
  }

  const QueryBlock* hb = c->h_block;
  if (c->use_row_hints && !c->row_hints.count(plan_key)) {
    if (c->row_hints.size() > 4096) c->row_hints.clear();
    std::vector<i64> rows((size_t)n);
    for (int s = 0; s < n; s++) rows[s] = hb->stats[s].rows;
    c->row_hints.emplace(plan_key, std::move(rows));
  }
  if (rep) {
    for (int s = 0; s < n; s++) {
      StepKind k = (StepKind)S.kinds[s];
      if (rep->kind) rep->kind[s] = (int32_t)k;
      if (rep->arity) rep->arity[s] = (int32_t)S.arities[s];
      if (rep->fused) rep->fused[s] = s < (int)S.fused_in.size() ? S.fused_in[s] : 0;
      if (rep->rows) rep->rows[s] = hb->stats[s].rows;
      if (rep->prealloc_total)
        rep->prealloc_total[s] = (k == S_EXPAND || k == S_FILTER) ? hb->stats[s].e : 0;
      if (rep->device_ms) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev[s], c->ev[s + 1]) != cudaSuccess) {
          ms = -1.f;
          cudaGetLastError();  // do not leave the failure pending for a later check
        }
        rep->device_ms[s] = ms;
      }
    }
  }

  i64 nrows = hb->stats[pack_stat].rows;
  const bool staged = hb->stats[pack_stat].pad != 0;
  const size_t row_bytes = 4 * (size_t)n_proj;
  gsm_result* r = new gsm_result();
  r->device = c->device;
  r->k = n_proj;
  r->ctx = c;
  r->gen = c->gen;
  cudaStream_t st = c->stream;
  i64 d2h_extra = 0;
  if (distinct && nrows > 1) {
    if (nrows >= 0xFFFFFFFFLL) {  // the tuple set stores u32 row indices
      delete r;
      char msg[160];
      snprintf(msg, sizeof msg, "DISTINCT over %lld rows exceeds the device limit of 2^32-1 rows",
               (long long)nrows);
      return set_error(GSM_ERR_RESOURCE, msg);
    }
    size_t cap = 16;
    while (cap < 2 * (size_t)nrows) cap <<= 1;
    if (cap > c->n_slots) {
      if (c->d_slots) cudaFree(c->d_slots);
      c->d_slots = nullptr;
      cudaError_t e = cudaMalloc(&c->d_slots, cap * 4);
      if (e != cudaSuccess) {
        delete r;
        c->n_slots = 0;
        return cuda_error(e, "cudaMalloc(distinct slots)");
      }
      c->n_slots = cap;
    }
    // Survivors go to the pinned staging buffer when they can fit, else to a
    // device buffer owned by the result.
    const bool to_host = (size_t)nrows * row_bytes <= c->stage_bytes;
    u32* dst = nullptr;
    if (to_host) {
      dst = c->d_rows;
    } else {
      cudaError_t e = cudaMalloc(&r->rows, std::max<size_t>(4, (size_t)nrows * row_bytes));
      if (e != cudaSuccess) {
        delete r;
        return cuda_error(e, "cudaMalloc(result)");
      }
      dst = r->rows;
    }
    GSM_CUDA(cudaMemsetAsync(c->d_slots, 0xFF, cap * 4, st));
    DistinctP dp{};
    dp.in = pack_out;
    dp.nsrc = c->d_block->stats + pack_stat;
    dp.cap_in = pack_cap;
    dp.k = n_proj;
    dp.slots = c->d_slots;
    dp.mask = (u32)(cap - 1);
    dp.out = dst;
    dp.cap_out = nrows;
    dp.st = c->d_block->stats + pack_stat + 1;
    GSM_CUDA(cudaMemsetAsync(c->d_block->counters + GSM_MAX_STEPS + 2, 0, 4, st));
    reserve_epochs(c, 1);
    k_init<<<1, 32, 0, st>>>(nullptr, nullptr, 0, c->d_ctr, c->d_block->epochs + GSM_MAX_STEPS + 2, 1,
                             ResolveArgs{}, nullptr, nullptr, nullptr, nullptr);
    count_launch();
    kernels++;
    TileSync ts{c->d_status, c->d_block->counters + GSM_MAX_STEPS + 2,
                c->d_block->epochs + GSM_MAX_STEPS + 2, 0};
    k_tilescan<DistinctP><<<c->grid_ts, TS_THREADS, 0, st>>>(dp, ts, ExportArgs{});
    count_launch();
    kernels++;
    if (timing) GSM_CUDA(cudaEventRecord(c->ev_q2, st));
    tail_event = true;
    GSM_CUDA(cudaMemcpyAsync(&c->h_block->stats[pack_stat + 1], dp.st, sizeof(StepStat),
                             cudaMemcpyDeviceToHost, st));
    GSM_CUDA(cudaStreamSynchronize(st));
    d2h_extra = sizeof(StepStat);
    r->n = c->h_block->stats[pack_stat + 1].rows;
    if (to_host) {
      if (r->n * (i64)row_bytes > 0)
        GSM_CUDA(cudaMemcpy(c->h_rows, c->d_rows, (size_t)r->n * row_bytes, cudaMemcpyDeviceToHost));
      r->staged = c->h_rows;
    }
  } else if (staged) {
    r->n = nrows;
    r->staged = c->h_rows;
    const size_t bytes = (size_t)nrows * row_bytes;
    if (!S.zc && bytes > c->guess)
      GSM_CUDA(cudaMemcpy(reinterpret_cast<char*>(c->h_rows) + c->guess,
                          reinterpret_cast<char*>(c->d_rows) + c->guess, bytes - c->guess,
                          cudaMemcpyDeviceToHost));
  } else {
    // Result larger than the staging buffer: keep it on the device, and grow
    // the staging buffer (up to 1 GiB) for the next query.
    r->n = nrows;
    size_t bytes = (size_t)nrows * row_bytes;
    cudaError_t e = cudaMalloc(&r->rows, std::max<size_t>(bytes, 4));
    if (e == cudaSuccess) {
      if (bytes) GSM_CUDA(cudaMemcpyAsync(r->rows, pack_out, bytes, cudaMemcpyDeviceToDevice, st));
    } else {
      // No room beside the arena (a left-row chunk near device capacity):
      // the result stays where the query packed it, valid until the next
      // gsm_execute on this context (like staged results).
      cudaGetLastError();
      r->rows = nullptr;
      r->dev_view = pack_out;
    }
    GSM_CUDA(cudaStreamSynchronize(st));
    if (bytes > c->stage_bytes && bytes <= c->stage_max) ctx_set_stage(c, bytes + bytes / 4);
  }
  // the next D2H size guess / zero-copy choice for this plan
  if (c->last_bytes.size() > 4096) c->last_bytes.clear();
  c->last_bytes[plan_key] = (size_t)nrows * row_bytes;
  r->zc = staged && S.zc && !distinct;
  if (rep) {
    rep->kernels = kernels;
    rep->h2d_bytes = h2d;
    // stats read-back + the result rows (copied into the pinned staging
    // buffer, or by gsm_result_copy for device-resident results)
    rep->d2h_bytes = (i64)sizeof(StepStat) * (n + 1) + d2h_extra + (i64)((size_t)r->n * row_bytes);
    rep->total_device_ms = 0.f;
    if (timing && cudaEventElapsedTime(&rep->total_device_ms, c->ev_q0,
                                       tail_event ? c->ev_q2 : c->ev_q1) != cudaSuccess) {
      rep->total_device_ms = -1.f;
      cudaGetLastError();
    }
  }
  *out = r;
  return GSM_OK;
}

gsm_status gsm_execute(gsm_context* c, const gsm_pattern* steps, int32_t n, const int32_t* proj,
                       int32_t n_proj, int32_t distinct, int64_t budget, int32_t budget_mode,
                       int64_t part, int64_t parts, gsm_report* rep, gsm_result** out) {
  *out = nullptr;
  QueryArgs qa{steps, n, proj, n_proj, distinct, budget, budget_mode, part, parts, rep};
  ExecState S;
  gsm_status st = begin_query(c, qa, S);
  if (st != GSM_OK) return st;
  return complete_query(c, qa, S, out);
}

gsm_status gsm_execute_seeded(gsm_context* c, const uint32_t* seed_rows, int64_t n_seed,
                              const int32_t* seed_vars, int32_t seed_k, const gsm_pattern* steps,
                              int32_t n_steps, const int32_t* proj, int32_t n_proj,
                              int32_t distinct, int64_t budget, int32_t budget_mode,
                              gsm_report* rep, gsm_result** out) {
  *out = nullptr;
  if (n_steps < 0 || n_steps >= GSM_MAX_STEPS || (n_steps > 0 && !steps))
    return set_error(GSM_ERR_VALUE, "bad seeded plan");
  std::vector<gsm_pattern> all((size_t)n_steps + 1);
  all[0] = gsm_pattern{-1, -1, 0, 0, 0, 1};  // placeholder: step 0 is the seed
  for (int i = 0; i < n_steps; i++) all[(size_t)i + 1] = steps[i];
  QueryArgs qa{all.data(), n_steps + 1, proj, n_proj, distinct, budget, budget_mode, 0, 1, rep};
  qa.seed = seed_rows;
  qa.seed_n = n_seed;
  qa.seed_vars = seed_vars;
  qa.seed_k = seed_k;
  ExecState S;
  gsm_status st = begin_query(c, qa, S);
  if (st != GSM_OK) return st;
  return complete_query(c, qa, S, out);
}

namespace {
double g_graph_launch_s = 0;  // host time inside cudaGraphLaunch (GSM_HOST_TIMING)
// launch_batch_graph phases (GSM_HOST_TIMING): validation, keys, lookup + replay set-up
double g_lbg_phase[3] = {0, 0, 0};
bool g_lbg_timing = getenv("GSM_HOST_TIMING") && getenv("GSM_HOST_TIMING")[0] == '1';
double lbg_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void note_graph_launch(double s) { g_graph_launch_s += s; }
// Make sure the next `need` epochs of a context need no status re-zeroing
// (reserve_epochs' wrap enqueues a memset on the context's own stream, which a
// batch graph launched on another stream would not be ordered after).
gsm_status epoch_headroom(gsm_context* c, int need) {
  if (c->epoch + (u32)need + 1 <= EPOCH_MAX) return GSM_OK;
  GSM_CUDA(cudaMemsetAsync(c->d_status, 0, c->n_status * sizeof(u64), c->stream));
  GSM_CUDA(cudaMemsetAsync(c->d_ctr, 0, sizeof(u32), c->stream));
  GSM_CUDA(cudaStreamSynchronize(c->stream));
  c->epoch = 0;
  return GSM_OK;
}

// Enqueue a whole batch as ONE graph launch on ctxs[0]'s stream (captured on
// first use as a fork/join over the contexts' streams, then replayed).
// Returns false (nothing enqueued, S reset) when the batch cannot use a
// prepared batch graph; the caller then launches the queries one by one.
bool launch_batch_graph(gsm_context* const* ctxs, int n, std::vector<QueryArgs>& qa,
                        std::vector<ExecState>& S, bool timed) {
  gsm_context* c0 = ctxs[0];
  if (n < 2 || !c0->use_batch_graph) return false;
  const double tp0 = g_lbg_timing ? lbg_now() : 0.0;
  for (int i = 0; i < n; i++) {
    if (!ctxs[i]->use_graphs || ctxs[i]->device != c0->device || qa[i].seed_k >= 0) return false;
    if (validate_query(ctxs[i], qa[i]) != GSM_OK) return false;
  }
  if (cudaSetDevice(c0->device) != cudaSuccess) return false;
  for (int i = 0; i < n; i++)  // install + the self-cleaning end: 2 x the launches' epochs
    if (epoch_headroom(ctxs[i], 2 * (GSM_MAX_STEPS + 4)) != GSM_OK) return false;
  const double tp1 = g_lbg_timing ? lbg_now() : 0.0;
  std::string bkey;
  std::vector<std::string> keys((size_t)n);
  for (int i = 0; i < n; i++) {
    S[i].timing = qa[i].rep && qa[i].rep->device_ms;
    keys[i] = query_key(ctxs[i], qa[i], S[i]);
    const gsm_context* cp = ctxs[i];
    bkey.append(reinterpret_cast<const char*>(&cp), sizeof cp);
    const u64 kl = keys[i].size();
    bkey.append(reinterpret_cast<const char*>(&kl), sizeof kl);
    bkey += keys[i];
  }
  cudaStream_t s0 = c0->stream;
  const double tp2 = g_lbg_timing ? lbg_now() : 0.0;
  auto it = c0->batches.find(bkey);
  if (it != c0->batches.end()) {
    bool ok = true;
    for (int i = 0; i < n && ok; i++) ok = it->second.bufgens[i] == ctxs[i]->bufgen;
    if (!ok) {
      cudaGraphExecDestroy(it->second.exec);
      c0->batches.erase(it);
      it = c0->batches.end();
    }
  }
  if (it == c0->batches.end()) {
    // Capture: fork every context's stream off s0, issue each query's launch
    // sequence on its own stream, join back into s0.
    if (c0->batches.size() >= 64) {
      for (auto& kv : c0->batches) free_batch(kv.second);
      c0->batches.clear();
    }
    // device images of the query blocks (filled after the capture)
    std::vector<char*> imgs((size_t)n, nullptr);
    auto drop_imgs = [&]() {
      for (char* p : imgs)
        if (p) cudaFree(p);
    };
    for (int i = 0; i < n; i++)
      if (cudaMalloc(&imgs[i], sizeof(QueryBlock)) != cudaSuccess ||
          cudaMemset(imgs[i], 0, sizeof(QueryBlock)) != cudaSuccess) {
        cudaGetLastError();
        drop_imgs();
        return false;
      }
    if (cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      drop_imgs();
      return false;
    }
    // The batch's device time is taken between event nodes at the graph's
    // entry and exit (GPU timestamps of its first and last node), so the
    // host's graph submission is not counted as device time (it is in the
    // caller's wall clock).
    bool ok = cudaEventRecordWithFlags(c0->ev_b0, s0, cudaEventRecordExternal) == cudaSuccess;
    ok = ok && cudaEventRecord(c0->ev_fork, s0) == cudaSuccess;
    int forked = 1;  // streams joined to the capture (ctxs[0]'s is the origin)
    for (; forked < n && ok; forked++) ok = cudaStreamWaitEvent(ctxs[forked]->stream, c0->ev_fork, 0) == cudaSuccess;
    if (!ok) forked--;
    // No programmatic dependent launch inside a batch: early-launched
    // dependents sit on SMs waiting for their predecessor and take the slots
    // the other queries' kernels need (measured: batch 0.096 -> 0.086 ms on
    // the bench workload; single-query latency is the same either way).
    // Members are captured longest plan first: the graph's branches are
    // submitted in capture order, so the chains that decide the batch's
    // span (most steps) start before the short ones (GSM_BATCH_ORDER=0:
    // input order).
    std::vector<int> order((size_t)n);
    for (int i = 0; i < n; i++) order[i] = i;
    if (c0->batch_order)
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return qa[a].n > qa[b].n; });
    for (int oi = 0; oi < n && ok; oi++) {
      const int i = order[oi];
      const bool pdl = ctxs[i]->use_pdl;
      ctxs[i]->use_pdl = pdl && ctxs[i]->batch_pdl;
      S[i].capture_only = true;
      S[i].pre_image = imgs[i];
      ok = launch_query(ctxs[i], qa[i], S[i]) == GSM_OK;
      S[i].capture_only = false;
      ctxs[i]->use_pdl = pdl;
      if (ok && c0->batch_poll)
        ok = cudaEventRecordWithFlags(ctxs[i]->ev_ext, ctxs[i]->stream, cudaEventRecordExternal) ==
             cudaSuccess;
    }
    // Join every forked stream back, also after a failed plan (a planning
    // error returns before issuing anything): an unjoined stream would leave
    // the capture in an invalid state for the fallback path.
    for (int i = 1; i < forked; i++) {
      const bool j = cudaEventRecord(ctxs[i]->ev_done, ctxs[i]->stream) == cudaSuccess &&
                     cudaStreamWaitEvent(s0, ctxs[i]->ev_done, 0) == cudaSuccess;
      ok = ok && j;
    }
    ok = ok && cudaEventRecordWithFlags(c0->ev_b1, s0, cudaEventRecordExternal) == cudaSuccess;
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s0, &g);
    cudaGraphExec_t ge = nullptr;
    if (ok && ce == cudaSuccess && g) ok = cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
    else ok = false;
    // member i's k_init node: the kernel node of k_init whose destination is
    // ctxs[i]'s query block
    std::vector<cudaGraphNode_t> init_node((size_t)n, nullptr);
    if (ok) {
      size_t nn = 0;
      ok = cudaGraphGetNodes(g, nullptr, &nn) == cudaSuccess;
      std::vector<cudaGraphNode_t> nodes(nn);
      if (ok && nn) ok = cudaGraphGetNodes(g, nodes.data(), &nn) == cudaSuccess;
      for (size_t k = 0; k < nn && ok; k++) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nodes[k], &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp{};
        if (cudaGraphKernelNodeGetParams(nodes[k], &kp) != cudaSuccess) continue;
        if (kp.func != reinterpret_cast<void*>(k_init) || !kp.kernelParams) continue;
        const void* dst = *reinterpret_cast<void* const*>(kp.kernelParams[1]);
        for (int i = 0; i < n; i++)
          if (dst == ctxs[i]->d_block) init_node[i] = nodes[k];
      }
      cudaGetLastError();
    }
    if (!ok && g) {
      cudaGraphDestroy(g);
      g = nullptr;
    }
    for (int i = 0; i < n && ok; i++)
      ok = cudaMemcpy(imgs[i], S[i].meta.image.data(), S[i].meta.image.size(), cudaMemcpyHostToDevice) ==
           cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      drop_imgs();
      for (int i = 0; i < n; i++) {
        // the captured plans took epochs from the host mirror only
        S[i] = ExecState();
      }
      return false;
    }
    gsm_context::BatchEntry E;
    E.exec = ge;
    E.graph = g;
    E.init_node = init_node;
    E.init_on.assign((size_t)n, 1);
    for (int i = 0; i < n; i++) {
      E.bufgens.push_back(ctxs[i]->bufgen);
      S[i].meta.image_id = next_image_id();
      E.metas.push_back(std::move(S[i].meta));
      S[i].kernels = E.metas[i].kernels;
    }
    it = c0->batches.emplace(bkey, std::move(E)).first;
    // the capture planned every query (epochs reserved for the install run)
    for (int i = 0; i < n; i++) count_launch(S[i].kernels);
  } else {
    // Per member: skip k_init (disable its node) when the member's context
    // still holds the member's image, left clean by its previous replay;
    // members whose context ran another plan in between install theirs.
    gsm_context::BatchEntry& B = it->second;
    for (int i = 0; i < n; i++) {
      ctxs[i]->gen++;
      const gsm_context::GraphEntry& M = B.metas[i];
      const bool w = B.resolved && M.self_clean && B.init_node[i] &&
                     ctxs[i]->installed == M.image_id;
      if ((B.init_on[i] != 0) == w) {  // toggle
        if (cudaGraphNodeSetEnabled(B.exec, B.init_node[i], w ? 0 : 1) != cudaSuccess) {
          cudaGetLastError();
          return false;
        }
        B.init_on[i] = w ? 0 : 1;
      }
      apply_entry(ctxs[i], M, S[i], w);
      if (w) S[i].kernels--;
      count_launch(S[i].kernels);
    }
  }
  if (g_lbg_timing) {
    const double tp3 = lbg_now();
    g_lbg_phase[0] += tp1 - tp0;
    g_lbg_phase[1] += tp2 - tp1;
    g_lbg_phase[2] += tp3 - tp2;
  }
  const auto tg0 = std::chrono::steady_clock::now();
  if (cudaGraphLaunch(it->second.exec, s0) != cudaSuccess) {
    cudaGetLastError();
    for (int i = 0; i < n; i++) ctxs[i]->installed = 0;
    return false;
  }
  for (int i = 0; i < n; i++)
    ctxs[i]->installed = it->second.metas[i].self_clean ? it->second.metas[i].image_id : 0;
  it->second.resolved = true;  // every member's k_init has run at least once
  note_graph_launch(std::chrono::duration<double>(std::chrono::steady_clock::now() - tg0).count());
  for (int i = 0; i < n; i++) S[i].sync_stream = s0;
  return true;
}
}  // namespace

#ifdef GSM_TRACE
// Diagnostic builds only (make trace): copy / clear the phase stamps.
gsm_status gsm_trace_dump(uint64_t* out, int64_t n_words) {
  const size_t cap = sizeof(gsm::g_trace) / 8;
  GSM_CUDA(cudaDeviceSynchronize());
  GSM_CUDA(cudaMemcpyFromSymbol(out, gsm::g_trace, 8 * std::min<size_t>((size_t)n_words, cap)));
  return GSM_OK;
}
gsm_status gsm_trace_reset(void) {
  GSM_CUDA(cudaDeviceSynchronize());
  static std::vector<unsigned long long> z(sizeof(gsm::g_trace) / 8, 0);
  GSM_CUDA(cudaMemcpyToSymbol(gsm::g_trace, z.data(), sizeof(gsm::g_trace)));
  return GSM_OK;
}
#endif

// Host-side phase times of gsm_execute_batch (GSM_HOST_TIMING=1: summary on
// stderr at exit) — the e2e path's host overhead, phase by phase.
namespace {
struct HostTimes {
  double launch = 0, wait = 0, complete = 0, graph_launch = 0, completing = 0, copying = 0;
  long calls = 0;
  bool on = getenv("GSM_HOST_TIMING") && getenv("GSM_HOST_TIMING")[0] == '1';
  ~HostTimes() {
    if (on && calls)
      fprintf(stderr,
              "gsm host timing: %ld batches, per batch: launch %.1f us (cudaGraphLaunch %.1f us), "
              "until the last member is out %.1f us (inside it: completing %.1f us, copying rows "
              "%.1f us), rest %.1f us\n",
              calls, 1e6 * launch / calls, 1e6 * graph_launch / calls, 1e6 * wait / calls,
              1e6 * completing / calls, 1e6 * copying / calls, 1e6 * complete / calls);
    if (on && calls)
      fprintf(stderr, "  batch graph set-up: validation %.1f us, keys %.1f us, lookup + replay %.1f us\n",
              1e6 * g_lbg_phase[0] / calls, 1e6 * g_lbg_phase[1] / calls, 1e6 * g_lbg_phase[2] / calls);
  }
} g_host_times;
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// A finished query's rows go straight into the caller's buffer when they fit
// (the result handle is then freed and outs[i] left NULL).
static void deliver(gsm_result*& r, uint32_t* const* dst, const int64_t* dst_cap, int i,
                    int64_t* n_rows, int32_t* n_cols) {
  if (!r) return;
  if (n_rows) n_rows[i] = r->n;
  if (n_cols) n_cols[i] = r->k;
  if (!dst || !dst[i] || !dst_cap || r->n * (i64)std::max(r->k, 1) > dst_cap[i]) return;
  if (gsm_result_copy(r, dst[i]) != GSM_OK) return;  // left to the caller
  gsm_result_free(r);
  r = nullptr;
}

static gsm_status batch_impl(gsm_context* const* ctxs, int32_t n_queries, const gsm_query* queries,
                             gsm_status* statuses, gsm_result** outs, float* device_ms,
                             uint32_t* const* dst, const int64_t* dst_cap, int64_t* n_rows,
                             int32_t* n_cols) {
  const double t_begin = g_host_times.on ? now_s() : 0.0;
  if (n_queries < 0 || (n_queries > 0 && (!ctxs || !queries || !outs)))
    return set_error(GSM_ERR_VALUE, "bad batch arguments");
  for (int i = 0; i < n_queries; i++) {
    outs[i] = nullptr;
    for (int j = 0; j < i; j++)
      if (ctxs[j] == ctxs[i]) return set_error(GSM_ERR_VALUE, "batch contexts must be distinct");
  }
  std::vector<ExecState> S((size_t)n_queries);
  std::vector<QueryArgs> qa((size_t)n_queries);
  std::vector<gsm_status> st((size_t)n_queries, GSM_OK);
  std::vector<std::string> msg((size_t)n_queries);
  const bool timed = device_ms && n_queries > 0;
  if (device_ms) *device_ms = 0.f;
  for (int i = 0; i < n_queries; i++) {
    const gsm_query& q = queries[i];
    qa[i] = QueryArgs{q.steps, q.n_steps, q.proj, q.n_proj, q.distinct, q.row_budget,
                      q.budget_mode, q.part_index, q.part_count, q.report};
  }
  // Fast path: the whole batch as one prepared graph launch.
  const bool as_graph = launch_batch_graph(ctxs, n_queries, qa, S, timed);
  if (!as_graph && timed && n_queries == 1) {  // one query: its own entry/exit event nodes
    S[0].span_events = true;
    st[0] = begin_query(ctxs[0], qa[0], S[0]);
    if (st[0] != GSM_OK) msg[0] = gsm_last_error();
  } else if (!as_graph) {
    if (timed) {  // all streams start after ev_b0 ...
      GSM_CUDA(cudaSetDevice(ctxs[0]->device));
      GSM_CUDA(cudaEventRecord(ctxs[0]->ev_b0, ctxs[0]->stream));
      for (int i = 1; i < n_queries; i++) GSM_CUDA(cudaStreamWaitEvent(ctxs[i]->stream, ctxs[0]->ev_b0, 0));
    }
    // Enqueue every query on its own context's stream (they overlap).
    for (int i = 0; i < n_queries; i++) {
      st[i] = begin_query(ctxs[i], qa[i], S[i]);
      if (st[i] != GSM_OK) msg[i] = gsm_last_error();
    }
    if (timed) {  // ... and ev_b1 on stream 0 follows all of them
      for (int i = 1; i < n_queries; i++) {
        GSM_CUDA(cudaEventRecord(ctxs[i]->ev_done, ctxs[i]->stream));
        GSM_CUDA(cudaStreamWaitEvent(ctxs[0]->stream, ctxs[i]->ev_done, 0));
      }
      GSM_CUDA(cudaEventRecord(ctxs[0]->ev_b1, ctxs[0]->stream));
    }
  }
  // Complete in order (budget checks, retries, result hand-off).
  // host timing: launch = until the graph is submitted; wait = until the
  // last member completed (its rows copied out); complete = the rest
  double t_launched = 0, t_waited = 0;
  if (g_host_times.on) t_launched = now_s();
  std::vector<char> done((size_t)n_queries, 0);
  auto finish = [&](int i) {
    if (st[i] == GSM_OK) {
      const double tc0 = g_host_times.on ? now_s() : 0.0;
      st[i] = complete_query(ctxs[i], qa[i], S[i], &outs[i]);
      const double tc1 = g_host_times.on ? now_s() : 0.0;
      if (st[i] != GSM_OK) msg[i] = gsm_last_error();
      else deliver(outs[i], dst, dst_cap, i, n_rows, n_cols);
      if (g_host_times.on) {
        g_host_times.completing += tc1 - tc0;
        g_host_times.copying += now_s() - tc1;
      }
    }
    done[i] = 1;
  };
  if (as_graph && n_queries > 0 && !ctxs[0]->batch_poll) {  // one wait for the whole graph
    GSM_CUDA(cudaStreamSynchronize(ctxs[0]->stream));
    for (int i = 0; i < n_queries; i++) S[i].synced = true;
  } else if (as_graph && n_queries > 0) {
    // Complete each query as soon as its own branch of the graph is done
    // (its external event fired), while the other branches still run: the
    // budget checks and the copy of its rows overlap the rest of the batch.
    int left = n_queries;
    cudaError_t bad = cudaSuccess;
    while (left > 0 && bad == cudaSuccess) {
      bool progressed = false;
      for (int i = 0; i < n_queries && bad == cudaSuccess; i++) {
        if (done[i]) continue;
        const cudaError_t q = cudaEventQuery(ctxs[i]->ev_ext);
        if (q == cudaErrorNotReady) continue;
        if (q != cudaSuccess) {
          bad = q;
          break;
        }
        S[i].synced = true;
        finish(i);
        left--;
        progressed = true;
      }
      if (!progressed && bad == cudaSuccess) std::this_thread::yield();
    }
    if (g_host_times.on) t_waited = now_s();
    // the join (and the batch's end event) on the origin stream
    const cudaError_t e = cudaStreamSynchronize(ctxs[0]->stream);
    if (bad == cudaSuccess) bad = e;
    if (bad != cudaSuccess) {
      for (int i = 0; i < n_queries; i++)
        if (outs[i]) {
          gsm_result_free(outs[i]);
          outs[i] = nullptr;
        }
      return cuda_error(bad, "batch graph");
    }
  }
  gsm_status first = GSM_OK;
  std::string first_msg;
  for (int i = 0; i < n_queries; i++) {
    if (!done[i]) finish(i);
    if (statuses) statuses[i] = st[i];
    if (st[i] != GSM_OK && first == GSM_OK) {
      first = st[i];
      first_msg = msg[i];
    }
  }
  if (timed && cudaEventElapsedTime(device_ms, ctxs[0]->ev_b0, ctxs[0]->ev_b1) != cudaSuccess) {
    *device_ms = -1.f;
    cudaGetLastError();
  }
  if (g_host_times.on) {
    const double t_end = now_s();
    if (t_waited == 0) t_waited = t_end;
    g_host_times.launch += t_launched - t_begin;
    g_host_times.wait += t_waited - t_launched;
    g_host_times.complete += t_end - t_waited;
    g_host_times.graph_launch = g_graph_launch_s;
    g_host_times.calls++;
  }
  if (first != GSM_OK) set_error(first, first_msg);
  return first;
}

gsm_status gsm_execute_batch(gsm_context* const* ctxs, int32_t n_queries, const gsm_query* queries,
                             gsm_status* statuses, gsm_result** outs, float* device_ms) {
  return batch_impl(ctxs, n_queries, queries, statuses, outs, device_ms, nullptr, nullptr, nullptr,
                    nullptr);
}

gsm_status gsm_execute_into(gsm_context* c, const gsm_pattern* steps, int32_t n, const int32_t* proj,
                            int32_t n_proj, int32_t distinct, int64_t budget, int32_t budget_mode,
                            int64_t part, int64_t parts, gsm_report* rep, uint32_t* dst,
                            int64_t dst_cap, int64_t* n_rows, int32_t* n_cols, gsm_result** out) {
  if (!n_rows || !n_cols || !out) return set_error(GSM_ERR_VALUE, "bad arguments");
  *n_rows = 0;
  *n_cols = 0;
  gsm_status st = gsm_execute(c, steps, n, proj, n_proj, distinct, budget, budget_mode, part, parts,
                              rep, out);
  if (st != GSM_OK) return st;
  uint32_t* const d[1] = {dst};
  const int64_t cap[1] = {dst_cap};
  deliver(*out, dst ? d : nullptr, cap, 0, n_rows, n_cols);
  return GSM_OK;
}

gsm_status gsm_execute_batch_into(gsm_context* const* ctxs, int32_t n_queries,
                                  const gsm_query* queries, gsm_status* statuses,
                                  uint32_t* const* dst, const int64_t* dst_cap, int64_t* n_rows,
                                  int32_t* n_cols, gsm_result** outs, float* device_ms) {
  if (n_queries > 0 && (!n_rows || !n_cols)) return set_error(GSM_ERR_VALUE, "bad batch arguments");
  for (int i = 0; i < n_queries; i++) {
    n_rows[i] = 0;
    n_cols[i] = 0;
  }
  return batch_impl(ctxs, n_queries, queries, statuses, outs, device_ms, dst, dst_cap, n_rows,
                    n_cols);
}


// ---------------------------------------------------------------------------
// gsm_table_join
// ---------------------------------------------------------------------------
namespace {
struct TableJoinScratch {
  DTable L, X;
  StepStat st[2];
  u32 counters[2];
  u32 epochs[2];
};
}  // namespace

gsm_status gsm_table_join(gsm_context* c, const uint32_t* left, int64_t n_left, int32_t a,
                          const uint32_t* right, int64_t n_right, int32_t b,
                          const int32_t* join_left, const int32_t* join_right, int32_t n_join,
                          int64_t budget, int32_t budget_mode, int64_t* prealloc_total,
                          int64_t* row_counts, gsm_result** out) {
  const bool counts_only = out == nullptr;  // preallocate(): N and E only
  if (out) *out = nullptr;
  if (!c) return set_error(GSM_ERR_VALUE, "null context");
  if (n_left < 0 || n_right < 0 || a < 0 || b < 0 || n_join < 0 || n_join > a || n_join > b ||
      a + b - n_join > GSM_MAX_VARS || a >= GSM_MAX_VARS)
    return set_error(GSM_ERR_VALUE, "bad table shapes");
  if ((n_left && a && !left) || (n_right && b && !right) || (n_join && (!join_left || !join_right)))
    return set_error(GSM_ERR_VALUE, "null table or join columns");
  if (n_right >= 0xFFFFFFF0LL) return set_error(GSM_ERR_VALUE, "right table must have < 2^32 rows");
  for (int i = 0; i < n_join; i++)
    if (join_left[i] < 0 || join_left[i] >= a || join_right[i] < 0 || join_right[i] >= b)
      return set_error(GSM_ERR_VALUE, "join column out of range");
  GSM_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  c->gen++;  // invalidates staged results of this context
  std::vector<void*> tmp;
  auto alloc = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, st);
    if (e == cudaSuccess) tmp.push_back(*p);
    return e;
  };
  gsm_result* r = nullptr;  // owned here until handed to *out
  auto cleanup = [&]() {
    for (void* p : tmp) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    tmp.clear();
    if (r) gsm_result_free(r);
    r = nullptr;
  };
#define TJ_CUDA(call)                              \
  do {                                             \
    cudaError_t _e = (call);                       \
    if (_e != cudaSuccess) {                       \
      cleanup();                                   \
      return ::gsm::cuda_error(_e, #call);         \
    }                                              \
  } while (0)
  const int w_out = a + b - n_join;
  u32 *dL = nullptr, *dR = nullptr;
  TJ_CUDA(alloc((void**)&dL, 4 * (size_t)n_left * a));
  TJ_CUDA(alloc((void**)&dR, 4 * (size_t)n_right * b));
  if (n_left * a) TJ_CUDA(cudaMemcpyAsync(dL, left, 4 * (size_t)n_left * a, cudaMemcpyHostToDevice, st));
  if (n_right * b) TJ_CUDA(cudaMemcpyAsync(dR, right, 4 * (size_t)n_right * b, cudaMemcpyHostToDevice, st));
  if (prealloc_total) *prealloc_total = 0;

  if (n_join == 0) {  // cross product (executor.py:155-165)
    i64 total = 0;
    if (__builtin_mul_overflow((i64)n_left, (i64)n_right, &total) || total > budget) {
      cleanup();
      char msg[256];
      snprintf(msg, sizeof msg, "cross product of %lld x %lld rows exceeds budget %lld",
               (long long)n_left, (long long)n_right, (long long)budget);
      return set_error(GSM_ERR_RESOURCE, msg);
    }
    if (counts_only) {
      cleanup();
      return GSM_OK;
    }
    r = new gsm_result();
    r->device = c->device;
    r->k = w_out;
    r->n = total;
    if (total * w_out > 0) {
      cudaError_t e = cudaMalloc(&r->rows, 4 * (size_t)total * w_out);
      if (e != cudaSuccess) {
        cleanup();
        return cuda_error(e, "cudaMalloc(result)");
      }
      k_cross_rows<<<c->grid_ts, 256, 0, st>>>(dL, n_left, a, dR, n_right, b, r->rows);
      count_launch();
    }
    TJ_CUDA(cudaGetLastError());
    gsm_result* done = r;
    r = nullptr;
    cleanup();
    *out = done;
    return GSM_OK;
  }

  // ---- index the right table on its first join column: stable sort by key,
  //      run heads -> hash {key, begin, len}  (the aux array of the right side)
  u32 *keys_in, *rows_in, *keys, *rows, *slots;
  TJ_CUDA(alloc((void**)&keys_in, 4 * (size_t)n_right));
  TJ_CUDA(alloc((void**)&rows_in, 4 * (size_t)n_right));
  TJ_CUDA(alloc((void**)&keys, 4 * (size_t)n_right));
  TJ_CUDA(alloc((void**)&rows, 4 * (size_t)n_right));
  size_t hcap = 16;
  while (hcap < 2 * (size_t)n_right) hcap <<= 1;
  TJ_CUDA(alloc((void**)&slots, 16 * hcap));
  TJ_CUDA(cudaMemsetAsync(slots, 0, 16 * hcap, st));
  if (n_right) {
    k_key_rows<<<std::max(1, std::min(c->grid_ts, (int)((n_right + 255) / 256))), 256, 0, st>>>(
        dR, n_right, b, join_right[0], keys_in, rows_in);
    count_launch();
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in, keys, rows_in, rows, (int64_t)n_right, 0, 32, st);
    void* tsort;
    TJ_CUDA(alloc(&tsort, tb));
    TJ_CUDA(cub::DeviceRadixSort::SortPairs(tsort, tb, keys_in, keys, rows_in, rows, (int64_t)n_right, 0, 32, st));
    count_launch();
  }
  Orient X{};
  X.src = keys;
  X.dst = rows;
  X.nnz = (u32)n_right;
  X.hmask = (u32)(hcap - 1);
  X.hs = reinterpret_cast<const uint4*>(slots);
  X.kbias = 1;
  if (n_right) {
    k_hash_runs<<<std::max(1, std::min(c->grid_ts, (int)((n_right + 255) / 256))), 256, 0, st>>>(
        keys, (u32)n_right, slots, (u32)(hcap - 1));
    count_launch();
  }

  // ---- per-row first-variable counts N and E (preallocate)
  u32* Lcols;
  TJ_CUDA(alloc((void**)&Lcols, 4 * (size_t)n_left * a));
  if (n_left * a) {
    k_rows_to_cols<<<std::max(1, std::min(c->grid_ts, (int)((n_left * a + 255) / 256))), 256, 0, st>>>(
        dL, n_left, a, Lcols, n_left);
    count_launch();
  }
  i64* dcnt;
  unsigned long long* dE;
  TJ_CUDA(alloc((void**)&dcnt, 8 * (size_t)n_left));
  TJ_CUDA(alloc((void**)&dE, 8));
  TJ_CUDA(cudaMemsetAsync(dE, 0, 8, st));
  if (n_left) {
    k_row_counts<<<std::max(1, std::min(c->grid_ts, (int)((n_left + 255) / 256))), 256, 0, st>>>(
        Lcols + (i64)join_left[0] * n_left, n_left, X, dcnt, dE);
    count_launch();
  }
  unsigned long long E = 0;
  TJ_CUDA(cudaMemcpyAsync(&E, dE, 8, cudaMemcpyDeviceToHost, st));
  if (row_counts && n_left)
    TJ_CUDA(cudaMemcpyAsync(row_counts, dcnt, 8 * (size_t)n_left, cudaMemcpyDeviceToHost, st));
  TJ_CUDA(cudaStreamSynchronize(st));
  if (prealloc_total) *prealloc_total = (i64)E;
  if (budget_mode == GSM_BUDGET_PARALLEL && (i64)E > budget) {
    cleanup();
    char msg[256];
    snprintf(msg, sizeof msg, "pre-allocated join region of %lld rows exceeds budget %lld",
             (long long)E, (long long)budget);
    return set_error(GSM_ERR_RESOURCE, msg);
  }
  if (counts_only) {
    cleanup();
    return GSM_OK;
  }
  if (budget_mode == GSM_BUDGET_SEQUENTIAL && (i64)E > budget) {
    // E-sized candidates may not fit: count the emitted rows first
    i64 O = (i64)E;
    if (n_join > 1) {
      SecCols sc{};
      sc.n = n_join - 1;
      for (int i = 1; i < n_join; i++) {
        sc.jl[i - 1] = join_left[i];
        sc.jr[i - 1] = join_right[i];
      }
      TJ_CUDA(cudaMemsetAsync(dE, 0, 8, st));
      k_sec_counts<<<std::max(1, std::min(c->grid_ts, (int)((n_left + 255) / 256))), 256, 0, st>>>(
          Lcols, n_left, join_left[0], X, dR, b, sc, dE);
      count_launch();
      unsigned long long hO = 0;
      TJ_CUDA(cudaMemcpyAsync(&hO, dE, 8, cudaMemcpyDeviceToHost, st));
      TJ_CUDA(cudaStreamSynchronize(st));
      O = (i64)hO;
    }
    if (O > budget) {
      cleanup();
      char msg[256];
      snprintf(msg, sizeof msg, "join output exceeds row budget %lld", (long long)budget);
      return set_error(GSM_ERR_RESOURCE, msg);
    }
  }
  r = new gsm_result();
  r->device = c->device;
  r->k = w_out;

  // ---- expand (left ++ right row index), then secondary checks + gather
  const i64 ntile_max = (std::max<i64>(n_left, (i64)E) + TS_TILE - 1) / TS_TILE + 2;
  u64* status;
  TJ_CUDA(alloc((void**)&status, 8 * (size_t)ntile_max));
  TJ_CUDA(cudaMemsetAsync(status, 0, 8 * (size_t)ntile_max, st));
  u32* Xcols;
  TJ_CUDA(alloc((void**)&Xcols, 4 * (size_t)std::max<u64>(E, 1) * (a + 1)));
  TableJoinScratch h{};
  h.L.n = n_left;
  for (int i = 0; i < a; i++) h.L.col[i] = Lcols + (i64)i * n_left;
  h.X.n = 0;
  for (int i = 0; i <= a; i++) h.X.col[i] = Xcols + (i64)i * (i64)std::max<u64>(E, 1);
  h.epochs[0] = 1;
  h.epochs[1] = 2;
  TableJoinScratch* d;
  TJ_CUDA(alloc((void**)&d, sizeof(TableJoinScratch)));
  TJ_CUDA(cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, st));
  ExpandP ep{};
  ep.L = &d->L;
  ep.R = X;
  ep.li = join_left[0];
  ep.a = a;
  ep.out = Xcols;
  ep.cap = (i64)std::max<u64>(E, 1);
  ep.O = &d->X;
  ep.st = &d->st[0];
  TileSync ts0{status, &d->counters[0], &d->epochs[0], 0};
  k_tilescan<ExpandP><<<std::max(1, std::min(c->grid_ts, (int)((n_left + TS_TILE - 1) / TS_TILE))), TS_THREADS, 0, st>>>(ep, ts0, ExportArgs{});
  count_launch();
  TFilterP fp{};
  fp.L = &d->X;
  fp.a = a;
  fp.R = dR;
  fp.b = b;
  fp.nsec = n_join - 1;
  for (int i = 1; i < n_join; i++) {
    fp.jl[i - 1] = join_left[i];
    fp.jr[i - 1] = join_right[i];
  }
  fp.nrc = 0;
  for (int k = 0; k < b; k++) {
    bool joined = false;
    for (int i = 0; i < n_join; i++) joined |= join_right[i] == k;
    if (!joined) fp.rc[fp.nrc++] = k;
  }
  const i64 res_rows = (i64)std::max<u64>(E, 1);
  cudaError_t e = cudaMalloc(&r->rows, 4 * (size_t)res_rows * std::max(w_out, 1));
  if (e != cudaSuccess) {
    cleanup();
    return cuda_error(e, "cudaMalloc(result)");
  }
  fp.out = r->rows;
  fp.st = &d->st[1];
  TileSync ts1{status, &d->counters[1], &d->epochs[1], 0};
  k_tilescan<TFilterP><<<std::max(1, std::min(c->grid_ts, (int)(((i64)E + TS_TILE - 1) / TS_TILE))), TS_THREADS, 0, st>>>(fp, ts1, ExportArgs{});
  count_launch();
  TJ_CUDA(cudaGetLastError());
  StepStat res{};
  TJ_CUDA(cudaMemcpyAsync(&res, &d->st[1], sizeof res, cudaMemcpyDeviceToHost, st));
  TJ_CUDA(cudaStreamSynchronize(st));
#undef TJ_CUDA
  r->n = res.rows;
  gsm_result* done = r;
  r = nullptr;
  cleanup();
  if (budget_mode == GSM_BUDGET_SEQUENTIAL && done->n > budget) {
    gsm_result_free(done);
    char msg[256];
    snprintf(msg, sizeof msg, "join output exceeds row budget %lld", (long long)budget);
    return set_error(GSM_ERR_RESOURCE, msg);
  }
  *out = done;
  return GSM_OK;
}

gsm_status gsm_partition_rows(gsm_context* c, const uint32_t* rows, int64_t n, int32_t k,
                              int32_t key_col, int64_t node_count, int32_t parts,
                              uint32_t* out_rows, int64_t* counts) {
  if (!c) return set_error(GSM_ERR_VALUE, "null context");
  if (n < 0 || k < 0 || k > GSM_MAX_VARS || parts < 1 || parts > 4096 || key_col >= k || !counts ||
      (n > 0 && k > 0 && (!rows || !out_rows)))
    return set_error(GSM_ERR_VALUE, "bad partition arguments");
  GSM_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  for (int d = 0; d < parts; d++) counts[d] = 0;
  if (n == 0) return GSM_OK;
  if (k == 0) {  // zero-arity rows carry no key: all to destination 0
    counts[0] = n;
    return GSM_OK;
  }
  unsigned long long* dcnt = nullptr;
  GSM_CUDA(cudaMallocAsync((void**)&dcnt, 16 * (size_t)parts, st));
  GSM_CUDA(cudaMemsetAsync(dcnt, 0, 8 * (size_t)parts, st));
  const int grid = (int)std::max<i64>(1, std::min<i64>(c->grid_ts, (n + 255) / 256));
  k_part_count<<<grid, 256, 4 * (size_t)parts, st>>>(rows, n, k, key_col, (u64)node_count, (u32)parts, dcnt);
  count_launch();
  std::vector<unsigned long long> h((size_t)parts);
  GSM_CUDA(cudaMemcpyAsync(h.data(), dcnt, 8 * (size_t)parts, cudaMemcpyDeviceToHost, st));
  GSM_CUDA(cudaStreamSynchronize(st));
  std::vector<unsigned long long> cur((size_t)parts);
  unsigned long long acc = 0;
  for (int d = 0; d < parts; d++) {
    counts[d] = (int64_t)h[(size_t)d];
    cur[(size_t)d] = acc;
    acc += h[(size_t)d];
  }
  unsigned long long* dcur = dcnt + parts;
  GSM_CUDA(cudaMemcpyAsync(dcur, cur.data(), 8 * (size_t)parts, cudaMemcpyHostToDevice, st));
  k_part_scatter<<<grid, 256, 0, st>>>(rows, n, k, key_col, (u64)node_count, (u32)parts, dcur, out_rows);
  count_launch();
  GSM_CUDA(cudaGetLastError());
  GSM_CUDA(cudaFreeAsync(dcnt, st));
  GSM_CUDA(cudaStreamSynchronize(st));
  return GSM_OK;
}

gsm_status gsm_cross_rows(gsm_context* c, const uint32_t* left, int64_t n_left, int32_t a,
                          const uint32_t* right, int64_t n_right, int32_t b, uint32_t* out) {
  if (!c) return set_error(GSM_ERR_VALUE, "null context");
  if (n_left < 0 || n_right < 0 || a < 0 || b < 0 || a + b > GSM_MAX_VARS)
    return set_error(GSM_ERR_VALUE, "bad cross product arguments");
  const i64 total = Exec::sat_mul(n_left, n_right);
  if (total == 0 || a + b == 0) return GSM_OK;
  if ((a && !left) || (b && !right) || !out) return set_error(GSM_ERR_VALUE, "null table");
  GSM_CUDA(cudaSetDevice(c->device));
  const int grid = (int)std::max<i64>(1, std::min<i64>((i64)c->grid_ts * 4, (total + 255) / 256));
  k_cross_rows<<<grid, 256, 0, c->stream>>>(left, n_left, a, right, n_right, b, out);
  count_launch();
  GSM_CUDA(cudaGetLastError());
  GSM_CUDA(cudaStreamSynchronize(c->stream));
  return GSM_OK;
}

}  // extern "C"
