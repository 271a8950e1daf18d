// hostio.cuh -- host <-> device transfers of pageable user buffers.
//
// The API takes plain host pointers (numpy arrays, C buffers), which are
// pageable: cudaMemcpy stages them through one driver buffer at ~11 GB/s
// H2D and ~4-20 GB/s D2H (measured on the B200 box, 535 MB).  Here a buffer
// moves in 16 MB chunks through a ring of pinned slots: host threads copy
// chunk i+1 between the user buffer and a slot while the copy engine moves
// chunk i, so the transfer runs near the pinned DMA rate (~48 GB/s H2D,
// ~57 GB/s D2H) and the page faults of a freshly allocated destination are
// taken by several threads at once.  Already-pinned buffers and small ones
// go straight to cudaMemcpyAsync.
//
// Included inside paracut_b200.cu's anonymous namespace.

namespace hostio {

#ifndef PCB_HOSTIO_CHUNK_MB
#define PCB_HOSTIO_CHUNK_MB 16
#endif
#ifndef PCB_HOSTIO_THREADS
#define PCB_HOSTIO_THREADS 8
#endif
constexpr size_t CHUNK = (size_t)PCB_HOSTIO_CHUNK_MB << 20;
constexpr int SLOTS = 4;
constexpr int THREADS = PCB_HOSTIO_THREADS;
constexpr size_t DIRECT_BELOW = (size_t)4 << 20;

// Persistent worker threads that split one memcpy between them.
class CopyPool {
 public:
  CopyPool() {
    for (int t = 1; t < THREADS; ++t) th_.emplace_back([this, t] { worker(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // dst[0:len) = src[0:len), split over THREADS threads (caller is thread 0)
  void copy(void* dst, const void* src, size_t len) {
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = (char*)dst;
      src_ = (const char*)src;
      len_ = len;
      pending_ = THREADS - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void part(int t) {
    const size_t per = ((len_ + THREADS - 1) / THREADS + 4095) & ~(size_t)4095;
    const size_t lo = per * t;
    if (lo < len_) memcpy(dst_ + lo, src_ + lo, (lo + per < len_ ? per : len_ - lo));
  }
  void worker(int t) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      part(t);
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct Stage {
  std::mutex m;  // one staged transfer at a time per process
  void* slot[SLOTS] = {};
  CopyPool* pool = nullptr;
  bool ready = false;
  bool init() {
    if (ready) return true;
    for (int i = 0; i < SLOTS; ++i)
      if (cudaHostAlloc(&slot[i], CHUNK, cudaHostAllocPortable) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
      }
    pool = new CopyPool();  // lives for the process
    ready = true;
    return true;
  }
};

inline Stage& stage() {
  static Stage* s = new Stage();  // never destroyed: workers outlive static teardown
  return *s;
}

inline bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Synchronous with respect to the host: returns when dst holds the data
// (the stream is used for ordering after earlier work on it).
inline cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  Stage& S = stage();
  if (bytes < DIRECT_BELOW || is_pinned(src)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  std::lock_guard<std::mutex> lk(S.m);
  if (!S.init()) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  cudaEvent_t ev[SLOTS] = {};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < SLOTS && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  bool used[SLOTS] = {};
  size_t i = 0;
  for (size_t off = 0; off < bytes && e == cudaSuccess; off += CHUNK, ++i) {
    const int s = (int)(i % SLOTS);
    const size_t len = bytes - off < CHUNK ? bytes - off : CHUNK;
    if (used[s]) e = cudaEventSynchronize(ev[s]);
    if (e != cudaSuccess) break;
    S.pool->copy(S.slot[s], (const char*)src + off, len);
    e = cudaMemcpyAsync((char*)dst + off, S.slot[s], len, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(ev[s], st);
    used[s] = true;
  }
  const cudaError_t e2 = cudaStreamSynchronize(st);
  for (int k = 0; k < SLOTS; ++k)
    if (ev[k]) cudaEventDestroy(ev[k]);
  return e != cudaSuccess ? e : e2;
}

inline cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  Stage& S = stage();
  if (bytes < DIRECT_BELOW || is_pinned(dst)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  std::lock_guard<std::mutex> lk(S.m);
  if (!S.init()) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  cudaEvent_t ev[SLOTS] = {};
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < SLOTS && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
  const size_t nch = (bytes + CHUNK - 1) / CHUNK;
  auto issue = [&](size_t c) {
    const int s = (int)(c % SLOTS);
    const size_t off = c * CHUNK;
    const size_t len = bytes - off < CHUNK ? bytes - off : CHUNK;
    cudaError_t r = cudaMemcpyAsync(S.slot[s], (const char*)src + off, len,
                                    cudaMemcpyDeviceToHost, st);
    return r == cudaSuccess ? cudaEventRecord(ev[s], st) : r;
  };
  for (size_t c = 0; c < nch && c < (size_t)SLOTS && e == cudaSuccess; ++c) e = issue(c);
  for (size_t c = 0; c < nch && e == cudaSuccess; ++c) {
    const int s = (int)(c % SLOTS);
    const size_t off = c * CHUNK;
    const size_t len = bytes - off < CHUNK ? bytes - off : CHUNK;
    e = cudaEventSynchronize(ev[s]);
    if (e != cudaSuccess) break;
    S.pool->copy((char*)dst + off, S.slot[s], len);
    if (c + SLOTS < nch) e = issue(c + SLOTS);
  }
  const cudaError_t e2 = cudaStreamSynchronize(st);
  for (int k = 0; k < SLOTS; ++k)
    if (ev[k]) cudaEventDestroy(ev[k]);
  return e != cudaSuccess ? e : e2;
}

}  // namespace hostio
