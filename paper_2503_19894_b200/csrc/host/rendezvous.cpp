// Shared-memory rendezvous of the ranks of one box (rendezvous.hpp).
#include "rendezvous.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>

#include "tilesim/core.hpp"

namespace tilesim {

namespace {
constexpr uint64_t kMagic = 0x3176645a52475354ULL;  // "TSGRZdv1"
constexpr size_t kHeaderBytes = 128;
}  // namespace

struct ShmRendezvous::Header {
  std::atomic<uint64_t> magic;
  std::atomic<uint32_t> world;
  std::atomic<uint32_t> arrived;     // ranks inside the current barrier
  std::atomic<uint32_t> generation;  // completed barriers
  std::atomic<uint32_t> attached;    // ranks that mapped the segment
};
static_assert(sizeof(std::atomic<uint64_t>) == 8 && std::atomic<uint32_t>::is_always_lock_free,
              "lock-free atomics in shared memory");

ShmRendezvous::Header* ShmRendezvous::hdr() const { return static_cast<Header*>(base_); }

void ShmRendezvous::make_id(unsigned char id[128]) {
  std::random_device rd;
  const uint64_t r = (static_cast<uint64_t>(rd()) << 32) ^ rd() ^
                     static_cast<uint64_t>(std::chrono::steady_clock::now().time_since_epoch().count());
  std::memset(id, 0, 128);
  std::snprintf(reinterpret_cast<char*>(id), 128, "/tsg-%d-%016llx", static_cast<int>(getpid()),
                static_cast<unsigned long long>(r));
}

ShmRendezvous::ShmRendezvous(const unsigned char id[128], int rank, int world, size_t slot_bytes, double timeout_s)
    : rank_(rank), world_(world), slot_bytes_((slot_bytes + 63) & ~size_t{63}), timeout_s_(timeout_s) {
  if (world < 1 || rank < 0 || rank >= world) throw ConfigError("rendezvous: rank outside [0, world)");
  name_.assign(reinterpret_cast<const char*>(id), strnlen(reinterpret_cast<const char*>(id), 127));
  if (name_.size() < 2 || name_[0] != '/') throw ConfigError("rendezvous: malformed unique id");
  total_ = kHeaderBytes + slot_bytes_ * static_cast<size_t>(world);
  const auto t0 = std::chrono::steady_clock::now();
  auto expired = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s_;
  };
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw SimError("rendezvous: shm_open(" + name_ + ") failed: " + std::strerror(errno));
    if (ftruncate(fd, static_cast<off_t>(total_)) != 0) {
      close(fd);
      shm_unlink(name_.c_str());
      throw SimError("rendezvous: ftruncate failed");
    }
  } else {
    for (;;) {  // wait for rank 0 to create and size the segment
      fd = shm_open(name_.c_str(), O_RDWR, 0600);
      if (fd >= 0) {
        struct stat sb;
        if (fstat(fd, &sb) == 0 && static_cast<size_t>(sb.st_size) >= total_) break;
        close(fd);
        fd = -1;
      }
      if (expired()) throw SimError("rendezvous: timed out waiting for rank 0's segment " + name_);
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  base_ = mmap(nullptr, total_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (base_ == MAP_FAILED) {
    base_ = nullptr;
    if (rank == 0) shm_unlink(name_.c_str());
    throw SimError("rendezvous: mmap failed");
  }
  Header* h = hdr();
  if (rank == 0) {
    new (&h->world) std::atomic<uint32_t>(static_cast<uint32_t>(world));
    new (&h->arrived) std::atomic<uint32_t>(0);
    new (&h->generation) std::atomic<uint32_t>(0);
    new (&h->attached) std::atomic<uint32_t>(0);
    h->magic.store(kMagic, std::memory_order_release);
  } else {
    while (h->magic.load(std::memory_order_acquire) != kMagic) {
      if (expired()) throw SimError("rendezvous: segment " + name_ + " never initialised");
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (h->world.load() != static_cast<uint32_t>(world)) throw ConfigError("rendezvous: world size differs from rank 0's");
  }
  h->attached.fetch_add(1);
  barrier();  // everyone mapped: the name can go (the mappings stay)
  if (rank == 0) shm_unlink(name_.c_str());
}

ShmRendezvous::~ShmRendezvous() {
  if (base_) munmap(base_, total_);
}

void* ShmRendezvous::slot(int r) {
  if (r < 0 || r >= world_) throw ConfigError("rendezvous: slot index out of range");
  return static_cast<unsigned char*>(base_) + kHeaderBytes + slot_bytes_ * static_cast<size_t>(r);
}

void ShmRendezvous::barrier() {
  Header* h = hdr();
  const uint32_t gen = h->generation.load(std::memory_order_acquire);
  if (h->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(world_)) {
    h->arrived.store(0, std::memory_order_relaxed);
    h->generation.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0; h->generation.load(std::memory_order_acquire) == gen; ++spin) {
    if (spin < 2048) continue;
    sched_yield();
    if ((spin & 1023) == 0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s_)
      throw SimError("rendezvous: barrier timed out (a rank died or diverged)");
  }
}

}  // namespace tilesim
