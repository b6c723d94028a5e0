// lod_ingest.cu -- disk -> device batch feed.
//
// The reference streams SIM files (io.py:60-92: 16-byte records f32 x, y, z,
// u8 r, g, b, a -- byte-identical to the update path's record layout) through
// an O_DIRECT reader (io.py:218-290) and a reader thread + queue
// (BatchSource, io.py:340-413) into run_frame_updates.  Here one native
// reader thread reads batch after batch with O_DIRECT (page-cache bypass;
// buffered reads when the filesystem refuses it) straight into a ring of
// page-locked buffers, so a batch goes disk -> pinned RAM -> HBM by DMA with
// no host-side copy or conversion; the consumer stages batch k+1's H2D copy
// (lod_prefetch_records) while batch k updates.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/lod_b200.h"

namespace {

constexpr size_t kAlign = 4096;  // O_DIRECT offset / size / buffer alignment

struct Slot {
  uint8_t *buf = nullptr;   // allocation
  uint8_t *data = nullptr;  // its first 4 KiB-aligned byte: the batch
  bool pinned = false;
  int64_t n = 0;       // records in the slot
  int state = 0;       // 0 free, 1 filled, 2 handed to the consumer
  long long seq = -1;  // batch index
};

}  // namespace

struct LodSim {
  std::string path;
  int fd = -1;
  bool direct = false;
  uint64_t size = 0;
  int64_t batch_records = 0;
  size_t slot_bytes = 0;
  std::vector<Slot> slots;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false, eof = false;
  int error = 0;
  long long next_hand = 0;  // the next batch handed to the consumer
  uint64_t bytes_read = 0;
  double read_seconds = 0.0;  // summed over the reader threads

  // Reader thread `t` of `nthreads` reads batches t, t + nthreads, ... into
  // slot b % slots once the consumer has released that slot's previous batch:
  // several reads in flight keep the drive's queue busy (one 16 MB read at a
  // time left an NVMe drive at ~60 % of its sequential rate).
  int nthreads = 1, finished = 0;
  std::vector<std::thread> pool;

  void run(int tid) {
    const uint64_t batch_bytes = (uint64_t)batch_records * 16ull;
    int fdl = direct ? open(path.c_str(), O_RDONLY | O_DIRECT) : open(path.c_str(), O_RDONLY);
    bool dl = direct && fdl >= 0;
    if (fdl < 0) fdl = open(path.c_str(), O_RDONLY);
    for (long long b = tid;; b += nthreads) {
      const uint64_t off = (uint64_t)b * batch_bytes;
      if (off >= size || fdl < 0) break;
      Slot *sl = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu);
        Slot &cand = slots[(size_t)(b % (long long)slots.size())];
        cv.wait(lk, [&] { return stop || error || (cand.state == 0 && cand.seq < b); });
        if (stop || error) break;
        cand.state = 3;  // being filled
        sl = &cand;
      }
      const uint64_t want = std::min<uint64_t>(batch_bytes, size - off);
      const auto t0 = std::chrono::steady_clock::now();
      uint64_t got = 0;
      while (got < want) {
        // O_DIRECT: aligned offset (batch sizes are multiples of 4096 bytes),
        // size rounded up (a short read at end of file is fine)
        size_t req = (size_t)(want - got);
        if (dl) req = (req + kAlign - 1) / kAlign * kAlign;
        const ssize_t r = pread(fdl, sl->data + got, req, (off_t)(off + got));
        if (r < 0 && dl && got == 0) {  // the filesystem refused O_DIRECT: buffered from here on
          close(fdl);
          fdl = open(path.c_str(), O_RDONLY);
          dl = false;
          std::lock_guard<std::mutex> lk(mu);
          direct = false;
          if (fdl < 0) break;
          continue;
        }
        if (r <= 0) break;
        got += (uint64_t)r;
      }
      if (got > want) got = want;
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::lock_guard<std::mutex> lk(mu);
      read_seconds += dt;
      bytes_read += got;
      if (got < want || got % 16) error = LOD_E_ARG;  // truncated file (io.py: Truncated)
      sl->n = (int64_t)(got / 16);
      sl->seq = b;
      sl->state = 1;
      cv.notify_all();
      if (error) break;
    }
    if (fdl >= 0) close(fdl);
    std::lock_guard<std::mutex> lk(mu);
    if (++finished == nthreads) eof = true;
    cv.notify_all();
  }
};

extern "C" {

int lod_sim_open(const char *path, int64_t batch_records, int32_t slots, LodSim **out) {
  if (!path || !out || batch_records <= 0 || slots < 2) return LOD_E_ARG;
  struct stat st {};
  if (stat(path, &st) != 0) return LOD_E_ARG;
  if (st.st_size == 0 || st.st_size % 16) return LOD_E_ARG;  // io.py: EmptyFile / Truncated
  // batches of whole 4 KiB pages keep every O_DIRECT read aligned
  if ((batch_records * 16) % (int64_t)kAlign) return LOD_E_ARG;
  LodSim *s = new LodSim();
  s->path = path;
  s->size = (uint64_t)st.st_size;
  s->batch_records = batch_records;
  s->slot_bytes = (size_t)batch_records * 16 + 2 * kAlign;
#ifdef O_DIRECT
  s->fd = open(path, O_RDONLY | O_DIRECT);
  s->direct = s->fd >= 0;
#endif
  if (s->fd < 0) s->fd = open(path, O_RDONLY);
  if (s->fd < 0) {
    delete s;
    return LOD_E_ARG;
  }
  close(s->fd);  // each reader thread opens its own descriptor
  s->fd = -1;
  int ndev = 0;
  const bool gpu = cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
  cudaGetLastError();
  s->slots.resize((size_t)slots);
  for (auto &sl : s->slots) {
    void *p = nullptr;
    if (gpu && cudaHostAlloc(&p, s->slot_bytes, cudaHostAllocDefault) == cudaSuccess) {
      sl.pinned = true;  // page-locked: the H2D copy is a DMA (cudaHostAlloc is page aligned)
    } else {
      cudaGetLastError();
      if (posix_memalign(&p, kAlign, s->slot_bytes) != 0) p = nullptr;
    }
    if (!p) {
      for (auto &q : s->slots)
        if (q.buf) q.pinned ? (void)cudaFreeHost(q.buf) : free(q.buf);
      close(s->fd);
      delete s;
      return LOD_E_NOMEM;
    }
    sl.buf = static_cast<uint8_t *>(p);
    sl.data = sl.buf + ((kAlign - (uintptr_t)sl.buf % kAlign) % kAlign);
  }
  // reader threads: LOD_SIM_READERS (default 1), at most slots - 2 (the
  // consumer holds the batch updating and the one staged behind it).  On the
  // test box's drive one O_DIRECT reader streams 4.9 GB/s and six concurrent
  // ones 2.7 GB/s in total, so one is the default; striped / multi-device
  // volumes want more
  const char *env = getenv("LOD_SIM_READERS");
  s->nthreads = std::max(1, std::min(std::max(1, slots - 2), env ? atoi(env) : 1));
  for (int k = 0; k < s->nthreads; ++k) s->pool.emplace_back([s, k] { s->run(k); });
  *out = s;
  return LOD_OK;
}

// Next batch in file order (blocks until it is read); *n = 0 at end of file.
// The records stay valid until lod_sim_release(records).
int lod_sim_next(LodSim *s, const void **records, int64_t *n) {
  if (!s || !records || !n) return LOD_E_ARG;
  std::unique_lock<std::mutex> lk(s->mu);
  Slot &sl = s->slots[(size_t)(s->next_hand % (long long)s->slots.size())];
  s->cv.wait(lk, [&] { return (sl.state == 1 && sl.seq == s->next_hand) || s->eof || s->error; });
  if (!(sl.state == 1 && sl.seq == s->next_hand)) {
    *records = nullptr;
    *n = 0;
    return s->error;
  }
  sl.state = 2;
  ++s->next_hand;
  *records = sl.data;
  *n = sl.n;
  return LOD_OK;
}

int lod_sim_release(LodSim *s, const void *records) {
  if (!s || !records) return LOD_E_ARG;
  std::lock_guard<std::mutex> lk(s->mu);
  for (auto &sl : s->slots)
    if (sl.data == records && sl.state == 2) {
      sl.state = 0;
      s->cv.notify_all();
      return LOD_OK;
    }
  return LOD_E_ARG;
}

int lod_sim_info(LodSim *s, LodSimInfo *info) {
  if (!s || !info) return LOD_E_ARG;
  std::lock_guard<std::mutex> lk(s->mu);
  info->file_bytes = s->size;
  info->bytes_read = s->bytes_read;
  info->read_seconds = s->read_seconds;
  info->direct = s->direct ? 1 : 0;
  info->pinned = s->slots.empty() ? 0 : (s->slots[0].pinned ? 1 : 0);
  return LOD_OK;
}

int lod_sim_close(LodSim *s) {
  if (!s) return LOD_OK;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    s->stop = true;
    s->cv.notify_all();
  }
  for (auto &th : s->pool)
    if (th.joinable()) th.join();
  for (auto &sl : s->slots)
    if (sl.buf) sl.pinned ? (void)cudaFreeHost(sl.buf) : free(sl.buf);
  if (s->fd >= 0) close(s->fd);
  delete s;
  return LOD_OK;
}

}  // extern "C"
