// Host-side offload tiers of the executor: pinned DRAM (cudaHostAlloc, so
// every H2D/D2H is a DMA at full PCIe bandwidth) and a local NVMe file
// accessed with O_DIRECT through a small thread pool (queue depth = threads).
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace gs::engine {

constexpr uint64_t kNvmeAlign = 4096;
inline uint64_t align_down(uint64_t x, uint64_t a) { return x / a * a; }
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Pinned host buffer owner.
class PinnedArena {
 public:
  ~PinnedArena();
  // 4 KiB-aligned pinned allocation (cudaHostAlloc is page aligned), zeroed.
  uint8_t* alloc(uint64_t bytes);
  uint64_t bytes() const { return bytes_; }

 private:
  std::vector<void*> blocks_;
  uint64_t bytes_ = 0;
};

// Fixed pool of worker threads running std::function jobs.
class ThreadPool {
 public:
  // nice_incr > 0 lowers the workers' scheduling priority (setpriority)
  explicit ThreadPool(int n, int nice_incr = 0);
  ~ThreadPool();
  // Runs all jobs to completion on the pool (the caller blocks).
  void run_all(std::vector<std::function<void()>>& jobs);
  int size() const { return static_cast<int>(workers_.size()); }

 private:
  void loop();
  std::vector<std::thread> workers_;
  std::mutex call_mu_;  // one batch at a time per pool
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::function<void()>>* batch_ = nullptr;
  size_t next_ = 0, finished_ = 0;
  uint64_t generation_ = 0;
  bool stop_ = false;
};

// Minimal io_uring submission/completion queue over raw syscalls (liburing
// is not in the image): O_DIRECT reads / writes of fixed-size pieces with up
// to `depth` in flight.  One ring per direction; not thread-safe by itself.
class Uring {
 public:
  explicit Uring(unsigned depth);
  ~Uring();
  bool ok() const { return fd_ >= 0; }
  // Transfers [off, off + bytes) between the file and buf in `piece`-byte
  // requests, keeping the queue full; short transfers are resubmitted.
  // Returns an error string (empty on success).
  std::string transfer(int file_fd, bool write, uint64_t off, uint8_t* buf, uint64_t bytes, uint64_t piece);

 private:
  int fd_ = -1;
  unsigned depth_ = 0;
  void* sq_ptr_ = nullptr;
  void* cq_ptr_ = nullptr;
  void* sqes_ = nullptr;
  size_t sq_len_ = 0, cq_len_ = 0, sqes_len_ = 0;
  unsigned *sq_head_ = nullptr, *sq_tail_ = nullptr, *sq_mask_ = nullptr, *sq_array_ = nullptr;
  unsigned *cq_head_ = nullptr, *cq_tail_ = nullptr, *cq_mask_ = nullptr;
  void* cqes_ = nullptr;
};

// The NVMe tier: one preallocated file, regions handed out 4 KiB-aligned.
// Transfers are split into <= chunk-sized pieces issued concurrently —
// through io_uring (queue depth 32) when the kernel allows it, else on a
// small pread/pwrite thread pool (GS_NVME_URING=0 forces the pool).
class NvmeFile {
 public:
  NvmeFile(const std::string& dir, bool odirect, int threads);
  ~NvmeFile();
  // Reserves `bytes` (rounded up to 4 KiB); returns the file offset.
  uint64_t reserve(uint64_t bytes);
  void finalize_size();
  // Host buffer and file offset must be 4 KiB-aligned; bytes is rounded up
  // to 4 KiB (the padding lives inside the reservation).  Returns physical
  // bytes moved.
  uint64_t write(uint64_t off, const void* src, uint64_t bytes);
  uint64_t read(uint64_t off, void* dst, uint64_t bytes);
  const std::string& path() const { return path_; }
  bool direct() const { return direct_; }

 private:
  uint64_t io(bool write, uint64_t off, void* buf, uint64_t bytes);
  std::string path_;
  int fd_ = -1;
  bool direct_ = false;
  uint64_t size_ = 0;
  // separate pools / rings so the SSD_R and SSD_W queues (distinct
  // dispatcher threads, full-duplex device) never share a batch
  ThreadPool read_pool_, write_pool_;
  std::unique_ptr<Uring> read_ring_, write_ring_;
  std::mutex read_mu_, write_mu_;

 public:
  bool uring() const { return read_ring_ != nullptr; }
};

}  // namespace gs::engine
