#include "host_tiers.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <linux/io_uring.h>
#include <sys/mman.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstdlib>
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
  if (cudaHostAlloc(&p, n, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess || !p)
    throw offsim::InfeasibleError("pinned host allocation of " + std::to_string(n) + " bytes failed");
  std::memset(p, 0, n);
  blocks_.push_back(p);
  bytes_ += n;
  return static_cast<uint8_t*>(p);
}

ThreadPool::ThreadPool(int n, int nice_incr) {
  for (int i = 0; i < n; ++i)
    workers_.emplace_back([this, nice_incr] {
      // background workers yield the cores to the executor's dispatcher
      // threads (the compute dispatcher enqueues kernels back to back)
      if (nice_incr > 0) (void)setpriority(PRIO_PROCESS, static_cast<id_t>(syscall(SYS_gettid)), nice_incr);
      loop();
    });
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

// ------------------------------------------------------------------ io_uring
Uring::Uring(unsigned depth) : depth_(depth) {
  io_uring_params p{};
  fd_ = static_cast<int>(syscall(__NR_io_uring_setup, depth, &p));
  if (fd_ < 0) return;
  sq_len_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
  cq_len_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
  sqes_len_ = p.sq_entries * sizeof(io_uring_sqe);
  sq_ptr_ = mmap(nullptr, sq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_, IORING_OFF_SQ_RING);
  cq_ptr_ = mmap(nullptr, cq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_, IORING_OFF_CQ_RING);
  sqes_ = mmap(nullptr, sqes_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_, IORING_OFF_SQES);
  if (sq_ptr_ == MAP_FAILED || cq_ptr_ == MAP_FAILED || sqes_ == MAP_FAILED) {
    close(fd_);
    fd_ = -1;
    return;
  }
  auto at = [](void* base, unsigned off) { return reinterpret_cast<unsigned*>(static_cast<uint8_t*>(base) + off); };
  sq_head_ = at(sq_ptr_, p.sq_off.head);
  sq_tail_ = at(sq_ptr_, p.sq_off.tail);
  sq_mask_ = at(sq_ptr_, p.sq_off.ring_mask);
  sq_array_ = at(sq_ptr_, p.sq_off.array);
  cq_head_ = at(cq_ptr_, p.cq_off.head);
  cq_tail_ = at(cq_ptr_, p.cq_off.tail);
  cq_mask_ = at(cq_ptr_, p.cq_off.ring_mask);
  cqes_ = static_cast<uint8_t*>(cq_ptr_) + p.cq_off.cqes;
}

Uring::~Uring() {
  if (sq_ptr_ && sq_ptr_ != MAP_FAILED) munmap(sq_ptr_, sq_len_);
  if (cq_ptr_ && cq_ptr_ != MAP_FAILED) munmap(cq_ptr_, cq_len_);
  if (sqes_ && sqes_ != MAP_FAILED) munmap(sqes_, sqes_len_);
  if (fd_ >= 0) close(fd_);
}

std::string Uring::transfer(int file_fd, bool write, uint64_t off, uint8_t* buf, uint64_t bytes, uint64_t piece) {
  struct Req {
    uint64_t pos, len;
  };
  std::vector<Req> todo;
  for (uint64_t pos = 0; pos < bytes; pos += piece) todo.push_back({pos, std::min(piece, bytes - pos)});
  size_t next = 0;
  // Accounting from the rings themselves: the kernel advances the SQ head as
  // it consumes entries, so `queued - consumed` entries wait in the SQ and
  // `consumed - completed` requests are in flight, whatever io_uring_enter
  // returned.
  const unsigned head0 = __atomic_load_n(sq_head_, __ATOMIC_ACQUIRE);
  unsigned tail = __atomic_load_n(sq_tail_, __ATOMIC_RELAXED);
  unsigned completed = 0;
  std::string err;
  io_uring_sqe* sqes = static_cast<io_uring_sqe*>(sqes_);
  io_uring_cqe* cqes = static_cast<io_uring_cqe*>(cqes_);
  auto reap = [&] {
    unsigned head = __atomic_load_n(cq_head_, __ATOMIC_RELAXED);
    const unsigned ctail = __atomic_load_n(cq_tail_, __ATOMIC_ACQUIRE);
    for (; head != ctail; ++head) {
      const io_uring_cqe& c = cqes[head & *cq_mask_];
      ++completed;
      if (!err.empty()) continue;  // draining after an error
      const Req q = todo[static_cast<size_t>(c.user_data)];
      if (c.res < 0) err = std::string(write ? "write: " : "read: ") + std::strerror(-c.res);
      else if (c.res == 0) err = std::string(write ? "write" : "read") + ": unexpected EOF";
      else if (static_cast<uint64_t>(c.res) < q.len)  // short transfer: queue the rest
        todo.push_back({q.pos + static_cast<uint64_t>(c.res), q.len - static_cast<uint64_t>(c.res)});
    }
    __atomic_store_n(cq_head_, head, __ATOMIC_RELEASE);
  };
  for (;;) {
    const unsigned consumed = __atomic_load_n(sq_head_, __ATOMIC_ACQUIRE) - head0;
    const unsigned queued = tail - head0;
    const unsigned inflight = consumed - completed, waiting = queued - consumed;
    if (!err.empty()) {
      // stop issuing: withdraw entries the kernel has not consumed, then
      // drain the in-flight requests so no CQE outlives this call
      if (waiting) __atomic_store_n(sq_tail_, tail -= waiting, __ATOMIC_RELEASE);
      if (inflight == 0) return err;
      syscall(__NR_io_uring_enter, fd_, 0, 1, IORING_ENTER_GETEVENTS, nullptr, 0);
      reap();
      continue;
    }
    if (next >= todo.size() && inflight == 0 && waiting == 0) return {};
    while (next < todo.size() && (tail - head0) - completed < depth_) {
      const unsigned idx = tail & *sq_mask_;
      io_uring_sqe& e = sqes[idx];
      std::memset(&e, 0, sizeof(e));
      e.opcode = write ? IORING_OP_WRITE : IORING_OP_READ;
      e.fd = file_fd;
      e.addr = reinterpret_cast<uint64_t>(buf + todo[next].pos);
      e.len = static_cast<uint32_t>(todo[next].len);
      e.off = off + todo[next].pos;
      e.user_data = next;
      sq_array_[idx] = idx;
      ++tail;
      ++next;
    }
    __atomic_store_n(sq_tail_, tail, __ATOMIC_RELEASE);
    const unsigned to_submit = tail - __atomic_load_n(sq_head_, __ATOMIC_ACQUIRE);
    const long r = syscall(__NR_io_uring_enter, fd_, to_submit, 1, IORING_ENTER_GETEVENTS, nullptr, 0);
    if (r < 0 && errno != EINTR && errno != EAGAIN && errno != EBUSY)
      err = std::string("io_uring_enter: ") + std::strerror(errno);
    reap();
  }
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
  const char* e = getenv("GS_NVME_URING");
  if (!e || atoi(e) != 0) {
    read_ring_ = std::make_unique<Uring>(32);
    write_ring_ = std::make_unique<Uring>(32);
    if (!read_ring_->ok() || !write_ring_->ok()) {
      read_ring_.reset();
      write_ring_.reset();
    }
  }
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
  if (read_ring_) {
    std::lock_guard<std::mutex> g(wr ? write_mu_ : read_mu_);
    const std::string err =
        (wr ? write_ring_ : read_ring_)->transfer(fd_, wr, off, static_cast<uint8_t*>(buf), total, 2ull << 20);
    if (!err.empty()) throw std::runtime_error("NVMe tier (io_uring): " + err);
    return total;
  }
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
