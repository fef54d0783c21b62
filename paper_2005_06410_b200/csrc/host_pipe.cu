// host_pipe.cu -- the host-memory runtime behind cgb_conv_host.
//
// The reference entry points are synchronous calls on host buffers (conv.hpp:60-91);
// on B200 the cost of such a call is the PCIe traffic, not the kernel (≈0.6 ms of
// kernels against ≈15 ms of copies for the BASELINE workload). The batch is the
// outermost (slowest) dimension of both I (h x w x c x b) and O (k_n x h_o x w_o x b),
// so each image is one contiguous byte range on both sides; the runtime cuts the batch
// into chunks and runs
//
//     H2D(chunk k+1)  ||  conv(chunk k)  ||  D2H(chunk k-1)
//
// on three streams (H2D stream, the caller's compute stream, D2H stream), so the two
// PCIe directions and the tensor cores all run concurrently and the call costs about
// max(H2D bytes, D2H bytes) / link bandwidth plus one chunk of fill and drain.
//
// Pinned (page-locked) caller buffers are copied directly. Pageable buffers go through
// a ring of pinned bounce slots; the host-side copies into and out of the ring are
// split across a small persistent thread pool so they keep up with the link.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"

namespace cgb {

// ------------------------------------------------------------------ parallel memcpy pool
namespace {

// Persistent memcpy pool. A job is up to two (dst, src, n) segments cut into
// 1 MiB-aligned pieces that the caller and the workers claim with one 64-bit atomic
// holding (job generation << 32 | next piece), so a claim can only succeed for the job
// it was read for. Job descriptors are double-buffered by generation parity, and a
// descriptor is rewritten only when no thread is inside the job two generations back
// (active_ counts per slot, re-checked against the generation after entering): a late
// worker can never copy or count a piece of a job it did not claim from. Workers spin
// on the generation for a while before sleeping, so the per-job hand-off costs about a
// cache-line transfer rather than a futex wake-up.
class CopyPool {
 public:
  struct Seg {
    void* dst;
    const void* src;
    size_t n;
  };
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  // both segments copied when this returns (callers are serialised)
  void copy2(Seg a, Seg b) {
    const size_t total = a.n + b.n;
    if (total == 0) return;
    if (workers_.empty() || total < 2 * kPiece) {
      if (a.n) std::memcpy(a.dst, a.src, a.n);
      if (b.n) std::memcpy(b.dst, b.src, b.n);
      return;
    }
    std::lock_guard<std::mutex> caller(caller_mu_);
    const uint64_t g = ++gen_;  // caller-owned counter
    const int slot = (int)(g & 1);
    while (active_[slot].load(std::memory_order_acquire) != 0) cpu_relax();  // stragglers of job g - 2
    Job& j = jobs_[slot];
    j.seg[0] = a;
    j.seg[1] = b;
    const size_t parts = std::min<size_t>(4 * (workers_.size() + 1), (total + kPiece - 1) / kPiece);
    j.per = ((total + parts - 1) / parts + 4095) & ~size_t(4095);
    j.nparts = (uint32_t)((total + j.per - 1) / j.per);
    pending_.store((int)j.nparts, std::memory_order_relaxed);
    claim_.store(g << 32, std::memory_order_release);  // publishes the job
    if (sleepers_.load(std::memory_order_acquire) > 0) {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    work(g);
    while (pending_.load(std::memory_order_acquire) > 0) cpu_relax();
  }

 private:
  static constexpr size_t kPiece = size_t(1) << 20;
  struct Job {
    Seg seg[2] = {};
    size_t per = 0;
    uint32_t nparts = 0;
  };
  static void cpu_relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  CopyPool() {
    const int hw = (int)std::thread::hardware_concurrency();
    const int req = tuning().host_copy_threads;
    const int n = req > 0 ? req : std::min(8, std::max(1, hw / 2));
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { run(); });
  }
  ~CopyPool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    for (auto& t : workers_) t.join();
  }
  // claim and copy pieces of job g until none are left (or a newer job replaced it)
  void work(uint64_t g) {
    const int slot = (int)(g & 1);
    active_[slot].fetch_add(1, std::memory_order_acq_rel);
    if ((claim_.load(std::memory_order_acquire) >> 32) == g) {
      const Job& j = jobs_[slot];
      for (;;) {
        uint64_t c = claim_.load(std::memory_order_acquire);
        if ((c >> 32) != g || (uint32_t)c >= j.nparts) break;
        if (!claim_.compare_exchange_weak(c, c + 1, std::memory_order_acq_rel)) continue;
        size_t lo = (size_t)(uint32_t)c * j.per, hi = std::min(lo + j.per, j.seg[0].n + j.seg[1].n);
        for (int k = 0; k < 2 && lo < hi; ++k) {  // the piece may straddle the two segments
          const Seg& sg = j.seg[k];
          if (lo < sg.n) {
            const size_t e = std::min(hi, sg.n);
            std::memcpy(static_cast<char*>(sg.dst) + lo, static_cast<const char*>(sg.src) + lo, e - lo);
          }
          lo = lo > sg.n ? lo - sg.n : 0;
          hi = hi > sg.n ? hi - sg.n : 0;
        }
        pending_.fetch_sub(1, std::memory_order_acq_rel);
      }
    }
    active_[slot].fetch_sub(1, std::memory_order_release);
  }
  void run() {
    uint64_t seen = claim_.load(std::memory_order_acquire) >> 32;
    for (;;) {
      // spin ~100 us for the next job, then sleep
      for (int it = 0; it < 20000 && (claim_.load(std::memory_order_acquire) >> 32) == seen && !stop_.load(); ++it)
        cpu_relax();
      if ((claim_.load(std::memory_order_acquire) >> 32) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        sleepers_.fetch_add(1, std::memory_order_acq_rel);
        cv_.wait(lk, [&] { return stop_.load() || (claim_.load(std::memory_order_acquire) >> 32) != seen; });
        sleepers_.fetch_sub(1, std::memory_order_acq_rel);
      }
      if (stop_.load()) return;
      seen = claim_.load(std::memory_order_acquire) >> 32;
      work(seen);
    }
  }

  std::vector<std::thread> workers_;
  std::mutex mu_, caller_mu_;
  std::condition_variable cv_;
  Job jobs_[2];
  uint64_t gen_ = 0;                    // last published job (caller only)
  std::atomic<uint64_t> claim_{0};      // (job generation << 32) | next piece index
  std::atomic<int> active_[2] = {{0}, {0}};  // threads inside a job of slot (generation & 1)
  std::atomic<int> pending_{0}, sleepers_{0};
  std::atomic<bool> stop_{false};
};

// Per-device pipeline state: the two copy streams, their events, the pinned ring.
struct DeviceState {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in = nullptr, ev_comp = nullptr, ev_end = nullptr;
  static constexpr int kSlots = 4;
  cudaEvent_t ev_slot_in[kSlots] = {}, ev_slot_out[kSlots] = {};
  std::vector<cudaEvent_t> ev_chunk;  // per-chunk "input landed" events (pinned input)
  char* pin = nullptr;  // [kSlots in][kSlots out] bounce slots
  size_t slot_bytes = 0;
  bool ok = false;
};

std::mutex g_mu;
std::vector<DeviceState> g_dev;

cudaError_t device_state(int dev, DeviceState** out) {
  if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
  DeviceState& d = g_dev[dev];
  if (!d.ok) {
    cudaError_t e;
    const unsigned fl = cudaEventDisableTiming;
    if ((e = cudaStreamCreateWithFlags(&d.h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&d.d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
    for (cudaEvent_t* ev : {&d.ev_start, &d.ev_in, &d.ev_comp, &d.ev_end})
      if ((e = cudaEventCreateWithFlags(ev, fl)) != cudaSuccess) return e;
    for (int i = 0; i < DeviceState::kSlots; ++i) {
      if ((e = cudaEventCreateWithFlags(&d.ev_slot_in[i], fl)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&d.ev_slot_out[i], fl)) != cudaSuccess) return e;
    }
    d.ok = true;
  }
  *out = &d;
  return cudaSuccess;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

int64_t host_chunk_items(size_t in_item, size_t out_item, int64_t items) {
  const size_t target = (size_t)std::max<int64_t>(1, tuning().host_chunk_kb) * 1024;
  const size_t per = std::max<size_t>(1, std::max(in_item, out_item));
  int64_t c = (int64_t)std::max<size_t>(1, target / per);
  c = std::max<int64_t>(c, (items + 63) / 64);  // at most 64 chunks
  return std::min(c, items);
}

static cudaError_t pipeline(DeviceState* d, const HostPipe& io, cudaStream_t compute, std::string* where) {
  cudaError_t e = cudaSuccess;
  const int64_t chunk = io.chunk_items > 0 ? std::min(io.chunk_items, io.items) : io.items;
  // Chunk plan: equal chunks of about `chunk` items (a size ramp at both ends to shrink
  // the exposed first H2D / last D2H measured no gain: the call is link-bound).
  std::vector<int64_t> start;  // first item of each chunk; start.back() == items
  {
    const int64_t n = (io.items + chunk - 1) / chunk;
    for (int64_t k = 0; k <= n; ++k) start.push_back(io.items * k / n);
  }
  const int64_t nchunks = (int64_t)start.size() - 1;
  const char* in_h = static_cast<const char*>(io.in_host);
  char* out_h = static_cast<char*>(io.out_host);
  char* in_d = static_cast<char*>(io.in_dev);
  const char* out_d = static_cast<const char*>(io.out_dev);
  const bool no_bounce = tuning().host_no_bounce != 0;
  const bool direct_in = is_pinned(io.in_host) || no_bounce;
  const bool direct_out = is_pinned(io.out_host) || no_bounce;
#define CGB_TRY(call, what)       \
  do {                            \
    if ((e = (call)) != cudaSuccess) { \
      *where = what;              \
      return e;                   \
    }                             \
  } while (0)
  // pinned bounce ring for pageable buffers
  if (!direct_in || !direct_out) {
    const size_t need = (size_t)chunk * std::max(io.in_item, io.out_item);
    if (d->slot_bytes < need) {
      if (d->pin) cudaFreeHost(d->pin);
      d->pin = nullptr;
      d->slot_bytes = 0;
      CGB_TRY(cudaHostAlloc(reinterpret_cast<void**>(&d->pin), 2 * DeviceState::kSlots * need,
                            cudaHostAllocPortable),
              "pinned bounce ring");
      d->slot_bytes = need;
    }
  }
  auto slot_in = [&](int j) { return d->pin + (size_t)j * d->slot_bytes; };
  auto slot_out = [&](int j) { return d->pin + (size_t)(DeviceState::kSlots + j) * d->slot_bytes; };
  CopyPool& pool = CopyPool::get();

  // The copy streams start after whatever the caller queued on the compute stream.
  CGB_TRY(cudaEventRecord(d->ev_start, compute), "event record");
  CGB_TRY(cudaStreamWaitEvent(d->h2d, d->ev_start, 0), "stream wait");
  CGB_TRY(cudaStreamWaitEvent(d->d2h, d->ev_start, 0), "stream wait");
  for (const HostPipe::Extra& x : io.extra)  // per-call operands (the filters) go first
    CGB_TRY(cudaMemcpyAsync(x.dev, x.host, x.bytes, cudaMemcpyDefault, d->h2d), "H2D operand");
  // Pinned input: every chunk's H2D is queued up front, one event per chunk, so the copy
  // engine never waits for the host to enqueue the next chunk's conv and D2H.
  if (direct_in) {
    while ((int64_t)d->ev_chunk.size() < nchunks) {
      cudaEvent_t ev;
      CGB_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event create");
      d->ev_chunk.push_back(ev);
    }
    for (int64_t k = 0; k < nchunks; ++k) {
      const size_t off = (size_t)start[k] * io.in_item, ib = (size_t)(start[k + 1] - start[k]) * io.in_item;
      CGB_TRY(cudaMemcpyAsync(in_d + off, in_h + off, ib, cudaMemcpyDefault, d->h2d), "H2D input");
      CGB_TRY(cudaEventRecord(d->ev_chunk[k], d->h2d), "event record");
    }
  }

  // Pageable buffers: in iteration k the host fills bounce slot k%S with input chunk k
  // and empties the same slot's output half (chunk k-S) in ONE parallel copy job, then
  // queues H2D(k), conv(k), D2H(k); the device runs S chunks behind the host.
  constexpr int S = DeviceState::kSlots;
  auto out_seg = [&](int64_t k) -> CopyPool::Seg {
    const int64_t i0 = start[k], n = start[k + 1] - i0;
    return {out_h + (size_t)i0 * io.out_item, slot_out((int)(k % S)), (size_t)n * io.out_item};
  };
  for (int64_t k = 0; k < nchunks; ++k) {
    const int j = (int)(k % S);
    const int64_t i0 = start[k], n = start[k + 1] - i0;
    const size_t ib = (size_t)n * io.in_item, ob = (size_t)n * io.out_item;
    // ---- host side of the bounce ring
    CopyPool::Seg seg_in{nullptr, nullptr, 0}, seg_out{nullptr, nullptr, 0};
    if (!direct_in) {
      if (k >= S) CGB_TRY(cudaEventSynchronize(d->ev_slot_in[j]), "bounce slot wait");
      seg_in = {slot_in(j), in_h + (size_t)i0 * io.in_item, ib};
    }
    if (!direct_out && k >= S) {
      CGB_TRY(cudaEventSynchronize(d->ev_slot_out[j]), "bounce slot wait");
      seg_out = out_seg(k - S);
    }
    pool.copy2(seg_in, seg_out);
    // ---- H2D (bounce ring; pinned input was queued above)
    if (!direct_in) {
      CGB_TRY(cudaMemcpyAsync(in_d + (size_t)i0 * io.in_item, slot_in(j), ib, cudaMemcpyHostToDevice, d->h2d),
              "H2D input");
      CGB_TRY(cudaEventRecord(d->ev_slot_in[j], d->h2d), "event record");
      CGB_TRY(cudaEventRecord(d->ev_in, d->h2d), "event record");
    }
    // ---- compute
    CGB_TRY(cudaStreamWaitEvent(compute, direct_in ? d->ev_chunk[k] : d->ev_in, 0), "stream wait");
    if ((e = io.compute(io.ctx, i0, n, compute)) != cudaSuccess) {
      *where = "conv";
      return e;
    }
    CGB_TRY(cudaEventRecord(d->ev_comp, compute), "event record");
    // ---- D2H
    CGB_TRY(cudaStreamWaitEvent(d->d2h, d->ev_comp, 0), "stream wait");
    CGB_TRY(cudaMemcpyAsync(direct_out ? out_h + (size_t)i0 * io.out_item : slot_out(j),
                            out_d + (size_t)i0 * io.out_item, ob, cudaMemcpyDefault, d->d2h),
            "D2H output");
    if (!direct_out) CGB_TRY(cudaEventRecord(d->ev_slot_out[j], d->d2h), "event record");
  }
  if (!direct_out)
    for (int64_t k = std::max<int64_t>(0, nchunks - S); k < nchunks; ++k) {
      CGB_TRY(cudaEventSynchronize(d->ev_slot_out[k % S]), "D2H output");
      pool.copy2(out_seg(k), {nullptr, nullptr, 0});
    }
  // join: the compute stream ends after the last D2H (the call is synchronous anyway)
  CGB_TRY(cudaEventRecord(d->ev_end, d->d2h), "event record");
  CGB_TRY(cudaStreamWaitEvent(compute, d->ev_end, 0), "stream wait");
  CGB_TRY(cudaEventRecord(d->ev_end, d->h2d), "event record");
  CGB_TRY(cudaStreamWaitEvent(compute, d->ev_end, 0), "stream wait");
  CGB_TRY(cudaStreamSynchronize(compute), "sync");
#undef CGB_TRY
  return cudaSuccess;
}

cudaError_t run_host_pipeline(const HostPipe& io, cudaStream_t compute, std::string* where) {
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  DeviceState* d = nullptr;
  if (e == cudaSuccess) e = device_state(dev, &d);
  if (e != cudaSuccess) {
    *where = "host pipeline setup";
    return e;
  }
  e = pipeline(d, io, compute, where);
  if (e != cudaSuccess) {  // never return with copies still reading/writing caller memory
    cudaStreamSynchronize(d->h2d);
    cudaStreamSynchronize(d->d2h);
    cudaStreamSynchronize(compute);
  }
  return e;
}

}  // namespace cgb
