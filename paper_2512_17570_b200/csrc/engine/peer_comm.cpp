#include "peer_comm.hpp"

#include <cuda.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <thread>

#include "kernels.h"

namespace gs::engine {

namespace {

constexpr int kMaxBufs = 32;

struct ShmRank {
  std::atomic<uint32_t> posted;  // handles below are valid
  std::atomic<uint32_t> opened;  // this rank has mapped every peer
  int nbuf;
  cudaIpcMemHandle_t flags;
  cudaIpcMemHandle_t bufs[kMaxBufs];
};
struct Shm {
  ShmRank r[kMaxPeers];
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "cross-process atomics");

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("peer comm: ") + what + ": " + cudaGetErrorString(e));
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
// stream wait-value (a front-end semaphore acquire: no SM is held while a
// peer is behind) when the driver provides it; else the spin kernel
std::atomic<WaitFn> g_wait_fn{nullptr};
WaitFn wait_value_fn() {
  static bool probed = false;
  if (probed) return g_wait_fn.load();
  probed = true;
  WaitFn fn = nullptr;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    fn = reinterpret_cast<WaitFn>(p);
  (void)cudaGetLastError();
  g_wait_fn.store(fn);
  return fn;
}

template <typename Pred>
void poll(Pred pred, const char* what) {
  const auto t0 = std::chrono::steady_clock::now();
  while (!pred()) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(180))
      throw std::runtime_error(std::string("peer comm: timed out waiting for the other ranks to ") + what);
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

}  // namespace

std::vector<uint8_t> peer_comm_unique_id() {
  std::vector<uint8_t> id(128, 0);
  std::random_device rd;
  for (auto& b : id) b = static_cast<uint8_t>(rd());
  id[0] = 'g';
  id[1] = 's';
  return id;
}

PeerComm::PeerComm(int rank, int world, const std::vector<uint8_t>& id, int device)
    : rank_(rank), world_(world), device_(device) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    throw std::invalid_argument("peer comm: 1 <= world <= 8 and 0 <= rank < world required");
  if (id.size() != 128) throw std::invalid_argument("peer comm: the job id must be 128 bytes");
  check(cudaSetDevice(device), "cudaSetDevice");
  check(cudaMalloc(&flags_, sizeof(uint32_t) * kKinds * world), "cudaMalloc counters");
  check(cudaMemset(flags_, 0, sizeof(uint32_t) * kKinds * world), "memset counters");
  char name[64];
  uint64_t h = 1469598103934665603ull;  // FNV-1a of the id
  for (uint8_t b : id) h = (h ^ b) * 1099511628211ull;
  std::snprintf(name, sizeof name, "/gs_peer_%016llx", static_cast<unsigned long long>(h));
  shm_name_ = name;
  if (world_ == 1) return;
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw std::runtime_error("peer comm: shm_open failed");
  shm_bytes_ = sizeof(Shm);
  if (ftruncate(fd, static_cast<off_t>(shm_bytes_)) != 0) {
    close(fd);
    throw std::runtime_error("peer comm: ftruncate failed");
  }
  shm_ = mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (shm_ == MAP_FAILED) {
    shm_ = nullptr;
    throw std::runtime_error("peer comm: mmap failed");
  }
}

PeerComm::~PeerComm() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  if (flags_) cudaFree(flags_);
  if (shm_) {
    munmap(shm_, shm_bytes_);
    if (rank_ == 0) shm_unlink(shm_name_.c_str());
  }
}

int PeerComm::add(void* base) {
  if (connected_) throw std::logic_error("peer comm: add() after connect()");
  if (static_cast<int>(bufs_.size()) >= kMaxBufs) throw std::logic_error("peer comm: too many buffers");
  bufs_.push_back(base);
  return static_cast<int>(bufs_.size()) - 1;
}

void PeerComm::connect() {
  const int nb = static_cast<int>(bufs_.size());
  ptrs_.assign(static_cast<size_t>(nb) * world_, nullptr);
  peer_flags_.assign(static_cast<size_t>(world_), nullptr);
  for (int b = 0; b < nb; ++b) ptrs_[static_cast<size_t>(b) * world_ + rank_] = bufs_[static_cast<size_t>(b)];
  peer_flags_[static_cast<size_t>(rank_)] = flags_;
  if (world_ > 1) {
    Shm& sh = *static_cast<Shm*>(shm_);
    ShmRank& me = sh.r[rank_];
    me.nbuf = nb;
    check(cudaIpcGetMemHandle(&me.flags, flags_), "cudaIpcGetMemHandle (counters)");
    for (int b = 0; b < nb; ++b) check(cudaIpcGetMemHandle(&me.bufs[b], bufs_[static_cast<size_t>(b)]), "cudaIpcGetMemHandle");
    me.posted.store(1, std::memory_order_release);
    poll([&] {
      for (int r = 0; r < world_; ++r)
        if (sh.r[r].posted.load(std::memory_order_acquire) != 1) return false;
      return true;
    }, "post their IPC handles");
    for (int r = 0; r < world_; ++r) {
      if (r == rank_) continue;
      if (sh.r[r].nbuf != nb) throw std::runtime_error("peer comm: ranks registered different buffer counts");
      void* p = nullptr;
      check(cudaIpcOpenMemHandle(&p, sh.r[r].flags, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle (counters)");
      opened_.push_back(p);
      peer_flags_[static_cast<size_t>(r)] = static_cast<uint32_t*>(p);
      for (int b = 0; b < nb; ++b) {
        check(cudaIpcOpenMemHandle(&p, sh.r[r].bufs[b], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        opened_.push_back(p);
        ptrs_[static_cast<size_t>(b) * world_ + r] = p;
      }
    }
    me.opened.store(1, std::memory_order_release);
    poll([&] {
      for (int r = 0; r < world_; ++r)
        if (sh.r[r].opened.load(std::memory_order_acquire) != 1) return false;
      return true;
    }, "map the IPC handles");
  }
  connected_ = true;
}

void PeerComm::signal(cudaStream_t st, Kind kind, uint32_t value) {
  PeerFlags f{};
  for (int r = 0; r < world_; ++r) f.p[r] = peer_flags_[static_cast<size_t>(r)] + kind * world_ + rank_;
  check(gs::peer_signal(f, world_, value, st), "signal");
}

void PeerComm::wait(cudaStream_t st, Kind kind, uint32_t value) {
  if (world_ == 1) return;
  WaitFn fn = wait_value_fn();
  int r = 0;
  for (; fn && r < world_; ++r) {
    if (r == rank_) continue;
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(flags_ + kind * world_ + r);
    if (fn(reinterpret_cast<CUstream>(st), a, value, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
      g_wait_fn.store(nullptr);  // unsupported here: spin kernels from now on
      break;
    }
  }
  if (r >= world_) return;
  PeerFlags f{};
  int n = 0;
  for (int q = r; q < world_; ++q)
    if (q != rank_) f.p[n++] = flags_ + kind * world_ + q;
  check(gs::peer_wait_spin(f, n, value, st), "wait");
}

}  // namespace gs::engine
