// Host-buffer gated MLP forward: the reference's array-in / array-out boundary
// (mlp.py:102 mlp_forward(x: ndarray) -> ndarray) with the PCIe transfers hidden
// behind the sparse products.
//
// Tokens are cut into chunks; chunk c's host->device copy runs on one copy stream,
// its two block-sparse launches on the caller's stream, its device->host copy on a
// second copy stream, so copy-in of c+1, compute of c and copy-out of c-1 overlap
// (the two DMA directions are independent engines). Three device slots for X and Y
// chunks, one for the intermediate G (compute is serial on the caller's stream).
#include <mutex>
#include <vector>

#include "host.hpp"

namespace blast {
namespace {

// Per-device copy streams and a reusable event pool. Re-recording a pooled event in a
// later call is safe: cudaStreamWaitEvent captures the event's state when it is enqueued.
// The device's mutex is held for a whole call (calls on one device share the streams).
struct CopyStreams {
  std::mutex mu;
  cudaStream_t in = nullptr, out = nullptr;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t make() {
    if (next == pool.size()) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[next++];
  }
};

CopyStreams* copy_streams() {
  static std::mutex mu;
  static CopyStreams per_dev[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  CopyStreams& cs = per_dev[dev];
  if (!cs.in) {
    if (cudaStreamCreateWithFlags(&cs.in, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaStreamCreateWithFlags(&cs.out, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  }
  return &cs;
}

int64_t auto_chunk(int64_t m) {
  // ~5 middle chunks of 3/16 of the tokens plus first / last chunks of a third of that (the
  // exposed head: copy-in alone; tail: compute + copy-out alone). Chunks stay >= 512 tokens
  // so each still fills the 148 SMs. cfg3 (8192 tokens): 512 + 4 x 1536 + ... + 512 measured
  // 1.82 ms vs 1.89 ms for 1024-token chunks with 512-token ends (tools/pipe_tune.py).
  int64_t c = (m * 3 / 16 + 127) / 128 * 128;
  return std::max<int64_t>(c, 512);
}

}  // namespace
}  // namespace blast

using namespace blast;

extern "C" int blast_mlp_forward_host(const void* x_host, int64_t m, const blast_bcsc_t* gate,
                                      const blast_bcsc_t* up, const blast_bcsc_t* down,
                                      const blast_mlp_plan_t* plan, void* y_host,
                                      int64_t chunk_tokens, void* stream) {
  if (!gate || !up || !down) {
    set_error("invalid block-sparse matrix descriptor");
    return BLAST_EINVAL;
  }
  if (m < 0 || chunk_tokens < 0) {
    set_error("negative token count");
    return BLAST_EINVAL;
  }
  if (m == 0) return BLAST_OK;
  if (!x_host || !y_host) {
    set_error("mlp_forward_host: null host buffer");
    return BLAST_EINVAL;
  }
  const int64_t e = gate->rows, h = gate->cols;
  if (down->rows != h || down->cols != e) {
    set_error("gated MLP shape mismatch");
    return BLAST_EMISMATCH;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CopyStreams* cs = copy_streams();
  if (!cs) return cuda_status(cudaGetLastError(), "copy streams");
  const size_t elt = bytes_of(gate->dtype);
  const int64_t chunk = std::min<int64_t>(m, chunk_tokens ? chunk_tokens : auto_chunk(m));
  // chunk boundaries; the automatic schedule shortens the first and last chunks to a third,
  // the exposed head (copy-in alone) and tail (compute + copy-out alone)
  std::vector<int64_t> bounds{0};
  if (!chunk_tokens && m > 2 * chunk) {
    // (first / last chunk 512 tokens at cfg3: 1.796 ms vs 1.804 (384), 1.846 (256), 1.858
    // (128); profiles/r02/e2e_pipeline.txt)
    const int64_t half = std::max<int64_t>(128, chunk / 3 / 128 * 128);
    bounds.push_back(half);
    while (m - bounds.back() > half + chunk) bounds.push_back(bounds.back() + chunk);
    if (m - bounds.back() > half) bounds.push_back(m - half);
  } else {
    while (m - bounds.back() > chunk) bounds.push_back(bounds.back() + chunk);
  }
  bounds.push_back(m);
  const int64_t n_chunks = static_cast<int64_t>(bounds.size()) - 1;
  // X and Y slots: one per chunk while both fit 1 GiB (every copy-in is queued back to back
  // with no slot dependency), else three (copy-in may run two chunks ahead of the copy-out,
  // so neither DMA direction waits on the other through a shared slot)
  const size_t row_bytes = elt * e;
  const int slots = static_cast<int>(
      2 * static_cast<size_t>(n_chunks) * chunk * row_bytes <= (size_t(1) << 30)
          ? n_chunks
          : std::min<int64_t>(n_chunks, 3));

  Scratch sx, sy, sg;
  if (!sx.alloc(slots * chunk * row_bytes, st) || !sy.alloc(slots * chunk * row_bytes, st) ||
      !sg.alloc(chunk * h * elt, st))
    return cuda_status(cudaGetLastError(), "pipeline buffers");
  std::lock_guard<std::mutex> lock(cs->mu);
  cs->next = 0;
  CopyStreams& evs = *cs;
  cudaEvent_t ev_start = evs.make();
  if (!ev_start) return cuda_status(cudaGetLastError(), "event");
  cudaEventRecord(ev_start, st);  // buffers allocated, caller's prior work ordered
  cudaStreamWaitEvent(cs->in, ev_start, 0);
  cudaStreamWaitEvent(cs->out, ev_start, 0);

  // every exit joins both copy streams back into st, so the stream-ordered frees of the
  // scratch buffers follow all their uses
  auto join = [&](int rc) {
    for (cudaStream_t s : {cs->in, cs->out}) {
      cudaEvent_t e = evs.make();
      if (e) {
        cudaEventRecord(e, s);
        cudaStreamWaitEvent(st, e, 0);
      }
    }
    return rc;
  };
  std::vector<cudaEvent_t> ev_comp(n_chunks), ev_out(n_chunks);
  // BLAST_PIPE_TRACE=1 (diagnosis): per-chunk copy-in / compute / copy-out spans to stderr
  static const bool trace = [] {
    const char* e = getenv("BLAST_PIPE_TRACE");
    return e && e[0] == '1';
  }();
  std::vector<cudaEvent_t> tr;
  auto tmark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tr.push_back(e);
  };
  tmark(st);
  const char* xh = static_cast<const char*>(x_host);
  char* yh = static_cast<char*>(y_host);
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int slot = static_cast<int>(c % slots);
    const int64_t r0 = bounds[c], mc = bounds[c + 1] - r0;
    char* xd = sx.as<char>() + slot * chunk * row_bytes;
    char* yd = sy.as<char>() + slot * chunk * row_bytes;
    cudaEvent_t ev_in = evs.make();
    ev_comp[c] = evs.make();
    ev_out[c] = evs.make();
    if (!ev_in || !ev_comp[c] || !ev_out[c]) return join(cuda_status(cudaGetLastError(), "event"));
    // copy-in: the X slot is free once chunk c-slots' compute has consumed it
    if (c >= slots) cudaStreamWaitEvent(cs->in, ev_comp[c - slots], 0);
    tmark(cs->in);
    cudaError_t ce = cudaMemcpyAsync(xd, xh + r0 * row_bytes, mc * row_bytes,
                                     cudaMemcpyHostToDevice, cs->in);
    if (ce != cudaSuccess) return join(cuda_status(ce, "copy-in"));
    cudaEventRecord(ev_in, cs->in);
    tmark(cs->in);
    // compute: needs the chunk's X, and the Y slot drained by chunk c-slots' copy-out
    cudaStreamWaitEvent(st, ev_in, 0);
    if (c >= slots) cudaStreamWaitEvent(st, ev_out[c - slots], 0);
    tmark(st);
    int r = blast_mlp_forward(xd, mc, gate, up, down, plan, yd, nullptr, nullptr, sg.ptr, st);
    if (r) return join(r);
    cudaEventRecord(ev_comp[c], st);
    tmark(st);
    // copy-out
    cudaStreamWaitEvent(cs->out, ev_comp[c], 0);
    tmark(cs->out);
    ce = cudaMemcpyAsync(yh + r0 * row_bytes, yd, mc * row_bytes, cudaMemcpyDeviceToHost,
                         cs->out);
    if (ce != cudaSuccess) return join(cuda_status(ce, "copy-out"));
    cudaEventRecord(ev_out[c], cs->out);
    tmark(cs->out);
  }
  if (trace) {
    const int rc = join(check_launch("mlp_forward_host"));
    cudaStreamSynchronize(st);
    for (int64_t c = 0; c < n_chunks; ++c) {
      float t[6];
      for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&t[k], tr[0], tr[1 + 6 * c + k]);
      fprintf(stderr, "[blast pipe] chunk %lld (%lld tok): in %7.1f-%7.1f  mlp %7.1f-%7.1f  out %7.1f-%7.1f us\n",
              (long long)c, (long long)(bounds[c + 1] - bounds[c]), t[0] * 1e3, t[1] * 1e3,
              t[2] * 1e3, t[3] * 1e3, t[4] * 1e3, t[5] * 1e3);
    }
    for (cudaEvent_t e : tr) cudaEventDestroy(e);
    return rc;
  }
  // the caller's stream passes this point only after the last copy-out
  return join(check_launch("mlp_forward_host"));
}
