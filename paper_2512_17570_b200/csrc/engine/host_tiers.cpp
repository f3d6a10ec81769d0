#include "host_tiers.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <stdexcept>

#include "offsim/offsim.hpp"

namespace gs::engine {

PinnedArena::~PinnedArena() {
  for (void* p : blocks_) cudaFreeHost(p);
}

uint8_t* PinnedArena::alloc(uint64_t bytes) {
  if (bytes == 0) return nullptr;
  const uint64_t n = align_up(bytes, kNvmeAlign);
  void* p = nullptr;
  if (cudaHostAlloc(&p, n, cudaHostAllocPortable) != cudaSuccess || !p)
    throw offsim::InfeasibleError("pinned host allocation of " + std::to_string(n) + " bytes failed");
  std::memset(p, 0, n);
  blocks_.push_back(p);
  bytes_ += n;
  return static_cast<uint8_t*>(p);
}

ThreadPool::ThreadPool(int n) {
  for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop() {
  uint64_t seen = 0;
  for (;;) {
    std::function<void()>* job = nullptr;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || (batch_ && next_ < batch_->size()) || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
      if (!batch_ || next_ >= batch_->size()) continue;
      job = &(*batch_)[next_++];
    }
    (*job)();
    {
      std::lock_guard<std::mutex> g(mu_);
      ++finished_;
    }
    done_cv_.notify_all();
  }
}

void ThreadPool::run_all(std::vector<std::function<void()>>& jobs) {
  if (jobs.empty()) return;
  if (workers_.empty() || jobs.size() == 1) {
    for (auto& j : jobs) j();
    return;
  }
  std::lock_guard<std::mutex> call(call_mu_);
  std::unique_lock<std::mutex> lk(mu_);
  batch_ = &jobs;
  next_ = 0;
  finished_ = 0;
  ++generation_;
  cv_.notify_all();
  done_cv_.wait(lk, [&] { return finished_ == jobs.size(); });
  batch_ = nullptr;
}

NvmeFile::NvmeFile(const std::string& dir, bool odirect, int threads) : read_pool_(threads), write_pool_(threads) {
  std::string tmpl = dir + "/greedysnake_tier_XXXXXX";
  std::vector<char> buf(tmpl.begin(), tmpl.end());
  buf.push_back('\0');
  const int fd = mkstemp(buf.data());
  if (fd < 0) throw offsim::ValidationError("cannot create NVMe tier file in " + dir + ": " + std::strerror(errno));
  path_ = buf.data();
  close(fd);
  int flags = O_RDWR;
  if (odirect) flags |= O_DIRECT;
  fd_ = open(path_.c_str(), flags);
  direct_ = odirect;
  if (fd_ < 0 && odirect) {  // filesystem without O_DIRECT (tmpfs): buffered I/O
    fd_ = open(path_.c_str(), O_RDWR);
    direct_ = false;
  }
  if (fd_ < 0) throw offsim::ValidationError("cannot open NVMe tier file " + path_);
  unlink(path_.c_str());  // anonymous: space is released when the engine closes
}

NvmeFile::~NvmeFile() {
  if (fd_ >= 0) close(fd_);
}

uint64_t NvmeFile::reserve(uint64_t bytes) {
  const uint64_t off = size_;
  size_ += align_up(bytes, kNvmeAlign);
  return off;
}

void NvmeFile::finalize_size() {
  if (size_ == 0) return;
  if (posix_fallocate(fd_, 0, static_cast<off_t>(size_)) != 0 && ftruncate(fd_, static_cast<off_t>(size_)) != 0)
    throw offsim::InfeasibleError("cannot size NVMe tier file to " + std::to_string(size_) + " bytes");
}

uint64_t NvmeFile::io(bool wr, uint64_t off, void* buf, uint64_t bytes) {
  if (bytes == 0) return 0;
  const uint64_t total = align_up(bytes, kNvmeAlign);
  constexpr uint64_t kChunk = 8ull << 20;
  std::vector<std::function<void()>> jobs;
  std::mutex err_mu;
  std::string err;
  for (uint64_t pos = 0; pos < total; pos += kChunk) {
    const uint64_t n = std::min(kChunk, total - pos);
    jobs.emplace_back([=, this, &err, &err_mu] {
      uint64_t done = 0;
      while (done < n) {
        uint8_t* p = static_cast<uint8_t*>(buf) + pos + done;
        const off_t o = static_cast<off_t>(off + pos + done);
        const ssize_t r = wr ? pwrite(fd_, p, n - done, o) : pread(fd_, p, n - done, o);
        if (r <= 0) {
          if (r < 0 && errno == EINTR) continue;
          std::lock_guard<std::mutex> g(err_mu);
          err = std::string(wr ? "pwrite" : "pread") + " failed: " + (r < 0 ? std::strerror(errno) : "EOF");
          return;
        }
        done += static_cast<uint64_t>(r);
      }
    });
  }
  (wr ? write_pool_ : read_pool_).run_all(jobs);
  if (!err.empty()) throw std::runtime_error("NVMe tier: " + err);
  return total;
}

uint64_t NvmeFile::write(uint64_t off, const void* src, uint64_t bytes) {
  return io(true, off, const_cast<void*>(src), bytes);
}
uint64_t NvmeFile::read(uint64_t off, void* dst, uint64_t bytes) { return io(false, off, dst, bytes); }

}  // namespace gs::engine
