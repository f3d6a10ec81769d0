// Host-side offload tiers of the executor: pinned DRAM (cudaHostAlloc, so
// every H2D/D2H is a DMA at full PCIe bandwidth) and a local NVMe file
// accessed with O_DIRECT through a small thread pool (queue depth = threads).
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
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
  explicit ThreadPool(int n);
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

// The NVMe tier: one preallocated file, regions handed out 4 KiB-aligned.
// Transfers are split into <= chunk-sized pieces issued concurrently.
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
  // separate pools so the SSD_R and SSD_W queues (distinct dispatcher
  // threads, full-duplex device) never share a batch
  ThreadPool read_pool_, write_pool_;
};

}  // namespace gs::engine
