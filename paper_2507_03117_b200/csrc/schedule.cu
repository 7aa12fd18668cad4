// Cost-balanced static work distribution for the persistent tensor-core engine.
//
// A product's work items are (token tile t, output line j); every token tile of a line costs
// the same: the number of pipeline stages the line's plan holds. Round robin (item = cta +
// k * grid) hands each CTA a random mix of lines, and the per-CTA totals spread by ~10 %
// around the mean at cfg3 (profiles/r01/mma_side/cta_ends.txt), so the kernel ends with the
// slowest CTA. Here one small kernel computes a batched longest-processing-time assignment:
//
//   sequence: t-major, within a tile the lines in descending cost (ties by index);
//   batch k = the next `grid` items of the sequence; its largest item goes to the CTA with
//   the least accumulated cost, the second largest to the second least loaded, ...
//   (the lines are sorted once with a bitonic sort; a batch's items are ranked from their
//   sorted-run positions and two binary searches, its CTAs by counting; three barriers
//   per batch)
//
// Batches are consecutive slices of the t-major sequence, so the CTAs still sweep the token
// tiles together (the activation panels of the tiles in flight stay in L2), and CTA c's
// k-th item is sched[k * grid + c] (-1 in the last, partial batch). Any permutation of the
// items gives the same results bit for bit (each item computes its own output tile in a
// fixed order); the schedule only moves the kernel's end time.
#include <mutex>
#include <vector>

#include "host.hpp"

namespace blast {

constexpr int kSchedThreads = 1024;
constexpr int kSchedMaxLines = 8192;
constexpr int kSchedMaxGrid = 1024;

// cost of one item of line j, in quarter stages: 4 per pipeline stage + 3 for the item's
// accumulator hand-off and epilogue tail
__device__ __forceinline__ int line_cost(const int32_t* step_ptr, const int32_t* flags, int seq_gu,
                                         int j) {
  int stages;
  if (seq_gu) {
    const int fl = flags[j];
    stages = ((fl >> 2) & 0x7fff) + ((fl >> 17) & 0x7fff);
  } else {
    stages = step_ptr[j + 1] - step_ptr[j];
  }
  return 4 * stages + 3;
}

// ascending bitonic sort of n (power of two) 64-bit keys in shared memory, all threads
__device__ void bitonic_sort(unsigned long long* key, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = key[lo], b = key[hi];
        if ((a > b) == up) {
          key[lo] = b;
          key[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSchedThreads)
lpt_schedule_kernel(const int32_t* step_ptr, const int32_t* flags, int seq_gu, int n_lines,
                    int n_tiles, int grid, int pl, int pg, int32_t* out) {
  extern __shared__ unsigned long long sm[];
  unsigned long long* lkey = sm;         // [pl] lines by descending cost
  unsigned long long* ckey = lkey + pl;  // [pg] CTAs by ascending load
  int* order = reinterpret_cast<int*>(ckey + pg);  // [n_lines] line of sorted index i
  int* scost = order + n_lines;                    // [n_lines] its cost (descending)
  int* load = scost + n_lines;                     // [grid]
  int* item_at = load + grid;                      // [grid] batch item of rank k
  int* cta_at = item_at + grid;                    // [grid] CTA of rank k
  constexpr unsigned long long kMax = ~0ull;

  for (int j = threadIdx.x; j < pl; j += blockDim.x) {
    if (j < n_lines) {
      const int c = line_cost(step_ptr, flags, seq_gu, j);
      lkey[j] = (static_cast<unsigned long long>(0x7fffffff - c) << 32) | static_cast<unsigned>(j);
    } else {
      lkey[j] = kMax;
    }
  }
  for (int c = threadIdx.x; c < grid; c += blockDim.x) load[c] = 0;
  __syncthreads();
  bitonic_sort(lkey, pl);
  for (int i = threadIdx.x; i < n_lines; i += blockDim.x) {
    order[i] = static_cast<int>(lkey[i] & 0xffffffffu);
    scost[i] = 0x7fffffff - static_cast<int>(lkey[i] >> 32);
  }
  __syncthreads();

  const long long total = static_cast<long long>(n_tiles) * n_lines;
  const long long rows = (total + grid - 1) / grid;
  const unsigned L = static_cast<unsigned>(n_lines);
  for (long long r = 0; r < rows; ++r) {
    const long long p0 = r * grid;
    const int n = static_cast<int>(min(static_cast<long long>(grid), total - p0));
    // the batch = sequence positions [p0, p0 + n): one run of sorted indices per token tile
    // t_first .. t_last, the first starting at sorted index off0
    const long long t_first = p0 / n_lines;
    const unsigned off0 = static_cast<unsigned>(p0 - t_first * n_lines);
    const unsigned t_span = (off0 + static_cast<unsigned>(n) - 1u) / L;  // t_last - t_first
    // Rank of batch item k under the key (-cost, k): inside its own run the items ahead of it
    // are exactly the ones before it (a run is sorted by descending cost, ties by line = by
    // k); of an earlier run those with cost >= its cost, of a later run those with cost >.
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const unsigned q = off0 + static_cast<unsigned>(k);
      const unsigned tr = q / L, i = q - tr * L;  // tile (relative) and sorted index
      const int c = scost[i];
      int lo = 0, hi = n_lines;  // gt = #sorted lines with cost > c
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (scost[mid] > c) lo = mid + 1; else hi = mid;
      }
      const unsigned gt = static_cast<unsigned>(lo);
      hi = n_lines;  // ge = #sorted lines with cost >= c
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (scost[mid] >= c) lo = mid + 1; else hi = mid;
      }
      const unsigned ge = static_cast<unsigned>(lo);
      unsigned rank = i - (tr == 0 ? off0 : 0u);
      for (unsigned u = 0; u <= t_span; ++u) {
        if (u == tr) continue;
        const unsigned a = u == 0 ? off0 : 0u;
        const unsigned b = u == t_span ? off0 + static_cast<unsigned>(n) - u * L : L;
        const unsigned lim = u < tr ? ge : gt;
        rank += (lim < a ? a : lim > b ? b : lim) - a;
      }
      item_at[rank] = k;
    }
    for (int k = threadIdx.x; k < grid; k += blockDim.x)
      ckey[k] = (static_cast<unsigned long long>(load[k]) << 32) | static_cast<unsigned>(k);
    __syncthreads();
    // rank of every CTA by ascending load: four lanes per CTA count the smaller keys over a
    // quarter of the CTAs each (all keys distinct), summed with two shuffles
    for (int t4 = threadIdx.x; t4 < 4 * ((grid + 7) & ~7); t4 += blockDim.x) {
      const int c = t4 >> 2, part = t4 & 3;
      const bool valid = c < grid;
      const unsigned long long me = valid ? ckey[c] : 0ull;
      int rank = 0;
      if (valid) {
#pragma unroll 4
        for (int s2 = part; s2 < grid; s2 += 4) rank += ckey[s2] < me ? 1 : 0;
      }
      rank += __shfl_xor_sync(0xffffffffu, rank, 1);
      rank += __shfl_xor_sync(0xffffffffu, rank, 2);
      if (valid && part == 0) cta_at[rank] = c;
    }
    __syncthreads();
    // the k-th largest item of the batch to the k-th least loaded CTA
    for (int k = threadIdx.x; k < grid; k += blockDim.x) {
      const int cta = cta_at[k];
      int item = -1;
      if (k < n) {
        const unsigned q = off0 + static_cast<unsigned>(item_at[k]);
        const unsigned tr = q / L, i = q - tr * L;
        item = static_cast<int>((t_first + tr) * n_lines + order[i]);
        load[cta] += scost[i];
      }
      out[r * grid + cta] = item;
    }
    __syncthreads();
  }
}

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

static int launch_lpt_schedule(const int32_t* step_ptr, const int32_t* flags, int n_lines,
                               int n_tiles, int grid, bool seq_gu, int32_t* out, cudaStream_t st) {
  if (n_lines <= 0 || n_tiles <= 0 || grid <= 0) return BLAST_OK;
  if (n_lines > kSchedMaxLines || grid > kSchedMaxGrid) {
    set_error("schedule: at most %d lines and %d CTAs", kSchedMaxLines, kSchedMaxGrid);
    return BLAST_EINVAL;
  }
  const int pl = next_pow2(n_lines), pg = next_pow2(grid);
  const size_t smem = sizeof(unsigned long long) * (pl + pg) + sizeof(int) * (2 * n_lines + 3 * grid);
  static bool configured[64] = {};
  if (int rc = configure_smem(lpt_schedule_kernel, 160 * 1024, configured, "schedule smem attribute"))
    return rc;
  lpt_schedule_kernel<<<1, kSchedThreads, smem, st>>>(step_ptr, flags, seq_gu ? 1 : 0, n_lines,
                                                       n_tiles, grid, pl, pg, out);
  return check_launch("lpt_schedule");
}

namespace {
struct SchedEntry {
  const int32_t* step_ptr;
  const int32_t* flags;
  int n_lines, n_tiles, grid, seq_gu, dev;
  int32_t* buf;
  int rows;
  uint64_t last_use;
};
std::mutex g_sched_mu;
std::vector<SchedEntry> g_sched;
uint64_t g_sched_clock = 0;
constexpr size_t kSchedCacheMax = 128;
}  // namespace

// Returns the cached (or newly computed, stream-ordered) schedule for this plan and token
// tile count, or nullptr when round robin is used (one item per CTA or less, shapes beyond
// the scheduler's limits, BLAST_SCHEDULE=0, or a capture in progress with nothing cached).
// Entries are keyed by the plan's device pointers and shape; a plan rebuilt at the same
// address reuses a stale but still complete item permutation (correct, perhaps less
// balanced) until it ages out of the bounded cache.
const int32_t* balanced_schedule(const int32_t* step_ptr, const int32_t* flags, int n_lines,
                                 int n_tiles, int grid, bool seq_gu, cudaStream_t st,
                                 int* rows_out) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("BLAST_SCHEDULE");
    enabled = (e && e[0] == '0') ? 0 : 1;
  }
  const long long total = static_cast<long long>(n_tiles) * n_lines;
  if (!enabled || total <= grid || n_lines > kSchedMaxLines || grid > kSchedMaxGrid ||
      total > (1ll << 30))
    return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_sched_mu);
  for (auto& e : g_sched) {
    if (e.step_ptr == step_ptr && e.flags == flags && e.n_lines == n_lines &&
        e.n_tiles == n_tiles && e.grid == grid && e.seq_gu == static_cast<int>(seq_gu) &&
        e.dev == dev) {
      e.last_use = ++g_sched_clock;
      *rows_out = e.rows;
      return e.buf;
    }
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
    return nullptr;  // never allocate inside a graph capture
  const int rows = static_cast<int>((total + grid - 1) / grid);
  SchedEntry ent{step_ptr, flags, n_lines, n_tiles, grid, static_cast<int>(seq_gu), dev,
                 nullptr, rows, ++g_sched_clock};
  if (g_sched.size() >= kSchedCacheMax) {
    // evict the least recently used entry; freed in stream order on this stream
    auto it = std::min_element(g_sched.begin(), g_sched.end(),
                               [](const SchedEntry& a, const SchedEntry& b) {
                                 return a.last_use < b.last_use;
                               });
    cudaFreeAsync(it->buf, st);
    g_sched.erase(it);
  }
  retain_pool_memory();
  if (cudaMallocAsync(reinterpret_cast<void**>(&ent.buf), sizeof(int32_t) * rows * grid, st) !=
      cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (launch_lpt_schedule(step_ptr, flags, n_lines, n_tiles, grid, seq_gu, ent.buf, st) !=
      BLAST_OK) {
    cudaFreeAsync(ent.buf, st);
    return nullptr;
  }
  g_sched.push_back(ent);
  *rows_out = rows;
  return ent.buf;
}

}  // namespace blast

// Test / inspection entry: the schedule the engine would use, written to out[rows * grid]
// (rows = ceil(n_tiles * n_lines / grid)).
extern "C" int blast_balanced_schedule(const int32_t* step_ptr, const int32_t* flags,
                                       int32_t n_lines, int32_t n_tiles, int32_t grid,
                                       int32_t seq_gu, int32_t* out, void* stream) {
  return blast::launch_lpt_schedule(step_ptr, flags, n_lines, n_tiles, grid, seq_gu != 0, out,
                                    static_cast<cudaStream_t>(stream));
}
