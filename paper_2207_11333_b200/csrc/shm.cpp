// shm.cpp — one pinned copy of the Table-1 graph store shared by every rank of a node
// (SURVEY §8(e) "All ranks read one pinned, shared-memory copy of the store"
// "shuffled and disjointed subsets" read by every process; include/hgnn.h hg_store_create_shared).
// The creator validates the arrays (hg_store_create's checks), derives the per-edge slot and
// writes everything into a POSIX shared-memory object; other processes map it read-only.
// Either side can page-lock the mapping (cudaHostRegister) so collation reads pinned memory.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <new>
#include <string>

#include "hgnn.h"
#include "internal.h"

using namespace hg;

namespace {

constexpr char kMagic[8] = {'H', 'G', 'S', 'H', 'M', '0', '0', '1'};

struct ShmHead {  // followed by the arrays at the byte offsets below (64-byte aligned)
  char magic[8];
  int64_t G, N, E, total;
  int32_t F0, Fe, has_yn, max_nodes, max_deg, pad;
  int64_t no, eo, x, ea, y, yn, src, dst, slot;
};

int64_t a64(int64_t v) { return (v + 63) & ~int64_t(63); }

ShmHead layout(const hg_store *s) {
  ShmHead h{};
  std::memcpy(h.magic, kMagic, 8);
  h.G = s->G; h.N = s->N; h.E = s->E; h.F0 = s->F0; h.Fe = s->Fe; h.has_yn = s->yn != nullptr;
  h.max_nodes = s->max_nodes; h.max_deg = s->max_deg;
  int64_t p = a64(sizeof(ShmHead));
  h.no = p; p = a64(p + 8 * (s->G + 1));
  h.eo = p; p = a64(p + 8 * (s->G + 1));
  h.x = p; p = a64(p + 4 * s->N * s->F0);
  h.ea = p; p = a64(p + 4 * s->E * s->Fe);
  h.y = p; p = a64(p + 4 * s->G);
  h.yn = p; p = a64(p + (h.has_yn ? 4 * s->N : 0));
  h.src = p; p = a64(p + 4 * s->E);
  h.dst = p; p = a64(p + 4 * s->E);
  h.slot = p; p = a64(p + s->E);
  h.total = p;
  return h;
}

void adopt_mapping(hg_store *s, uint8_t *base, const ShmHead &h) {
  s->G = h.G; s->N = h.N; s->E = h.E; s->F0 = h.F0; s->Fe = h.Fe;
  s->max_nodes = h.max_nodes; s->max_deg = h.max_deg;
  s->no = reinterpret_cast<const int64_t *>(base + h.no);
  s->eo = reinterpret_cast<const int64_t *>(base + h.eo);
  s->x = reinterpret_cast<const float *>(base + h.x);
  s->ea = reinterpret_cast<const float *>(base + h.ea);
  s->y = reinterpret_cast<const float *>(base + h.y);
  s->yn = h.has_yn ? reinterpret_cast<const float *>(base + h.yn) : nullptr;
  s->src = reinterpret_cast<const int32_t *>(base + h.src);
  s->dst = reinterpret_cast<const int32_t *>(base + h.dst);
  s->slotp = base + h.slot;
}

hg_status pin(hg_store *s, int32_t want, unsigned flags) {
  if (!want) return HG_OK;
  const cudaError_t e = cudaHostRegister(s->shm_base, s->shm_bytes, flags);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HG_E_CUDA, "cudaHostRegister of the shared store: %s", cudaGetErrorString(e));
  }
  s->shm_pinned = true;
  return HG_OK;
}

}  // namespace

hg_store::~hg_store() {
  if (shm_base) {
    if (shm_pinned) cudaHostUnregister(shm_base);
    munmap(shm_base, shm_bytes);
  }
}

extern "C" {

hg_status hg_store_create_shared(const hg_store_desc *d, const char *name, int32_t pin_memory, int32_t threads,
                                 hg_store **out) {
  if (!d || !name || !out || name[0] != '/') return fail(HG_E_INVALID, "null argument or name not starting with '/'");
  *out = nullptr;
  hg_store *tmp = nullptr;
  hg_status st = hg_store_create(d, 0, threads, &tmp);  // validation + slot, borrowing the caller's arrays
  if (st) return st;
  const ShmHead h = layout(tmp);
  const int fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
  if (fd < 0) {
    hg_store_destroy(tmp);
    return fail(HG_E_IO, "shm_open(%s): %s", name, strerror(errno));
  }
  if (ftruncate(fd, h.total) != 0) {
    close(fd);
    shm_unlink(name);
    hg_store_destroy(tmp);
    return fail(HG_E_IO, "ftruncate(%s, %lld): %s", name, (long long)h.total, strerror(errno));
  }
  void *base = mmap(nullptr, h.total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (base == MAP_FAILED) {
    shm_unlink(name);
    hg_store_destroy(tmp);
    return fail(HG_E_IO, "mmap(%s): %s", name, strerror(errno));
  }
  uint8_t *b = static_cast<uint8_t *>(base);
  std::memcpy(b + h.no, tmp->no, 8 * (h.G + 1));
  std::memcpy(b + h.eo, tmp->eo, 8 * (h.G + 1));
  std::memcpy(b + h.x, tmp->x, 4 * h.N * h.F0);
  std::memcpy(b + h.ea, tmp->ea, 4 * h.E * h.Fe);
  std::memcpy(b + h.y, tmp->y, 4 * h.G);
  if (h.has_yn) std::memcpy(b + h.yn, tmp->yn, 4 * h.N);
  std::memcpy(b + h.src, tmp->src, 4 * h.E);
  std::memcpy(b + h.dst, tmp->dst, 4 * h.E);
  std::memcpy(b + h.slot, tmp->slotp, h.E);
  std::memcpy(b, &h, sizeof(h));  // the header last: a reader sees either no magic or a full store
  hg_store_destroy(tmp);
  hg_store *s = new (std::nothrow) hg_store();
  if (!s) {
    munmap(base, h.total);
    shm_unlink(name);
    return fail(HG_E_IO, "out of host memory");
  }
  s->shm_base = base;
  s->shm_bytes = (size_t)h.total;
  adopt_mapping(s, b, h);
  if ((st = pin(s, pin_memory, cudaHostRegisterDefault))) {
    delete s;
    shm_unlink(name);
    return st;
  }
  *out = s;
  return HG_OK;
}

hg_status hg_store_open_shared(const char *name, int32_t pin_memory, hg_store **out) {
  if (!name || !out) return fail(HG_E_INVALID, "null argument");
  *out = nullptr;
  const int fd = shm_open(name, O_RDONLY, 0);
  if (fd < 0) return fail(HG_E_IO, "shm_open(%s): %s", name, strerror(errno));
  struct stat sb;
  if (fstat(fd, &sb) != 0 || sb.st_size < (off_t)sizeof(ShmHead)) {
    close(fd);
    return fail(HG_E_IO, "%s: not a shared store (size)", name);
  }
  void *base = mmap(nullptr, sb.st_size, PROT_READ, MAP_SHARED, fd, 0);
  close(fd);
  if (base == MAP_FAILED) return fail(HG_E_IO, "mmap(%s): %s", name, strerror(errno));
  ShmHead h;
  std::memcpy(&h, base, sizeof(h));
  hg_store tmp_sizes;  // recompute the layout from the header's counts: it must match exactly
  tmp_sizes.G = h.G; tmp_sizes.N = h.N; tmp_sizes.E = h.E; tmp_sizes.F0 = h.F0; tmp_sizes.Fe = h.Fe;
  tmp_sizes.yn = h.has_yn ? reinterpret_cast<const float *>(1) : nullptr;
  const bool ok = std::memcmp(h.magic, kMagic, 8) == 0 && h.G >= 1 && h.N >= 0 && h.E >= 0 && h.F0 >= 1 &&
                  h.Fe >= 1 && h.total == (int64_t)sb.st_size && layout(&tmp_sizes).total == h.total;
  tmp_sizes.yn = nullptr;
  if (!ok) {
    munmap(base, sb.st_size);
    return fail(HG_E_IO, "%s: not a shared store (header)", name);
  }
  hg_store *s = new (std::nothrow) hg_store();
  if (!s) {
    munmap(base, sb.st_size);
    return fail(HG_E_IO, "out of host memory");
  }
  s->shm_base = base;
  s->shm_bytes = (size_t)sb.st_size;
  adopt_mapping(s, static_cast<uint8_t *>(base), h);
  hg_status st = pin(s, pin_memory, cudaHostRegisterReadOnly);
  if (st) {
    delete s;
    return st;
  }
  *out = s;
  return HG_OK;
}

hg_status hg_store_unlink_shared(const char *name) {
  if (!name) return fail(HG_E_INVALID, "null name");
  if (shm_unlink(name) != 0) return fail(HG_E_IO, "shm_unlink(%s): %s", name, strerror(errno));
  return HG_OK;
}

}  // extern "C"
