// container.cpp — on-disk packed graph container with subfiles,
// the ADIOS stand-in of PAPER.md:183-192: the Table-1 variables
// x, edge_index, edge_attr, y stored as global arrays with per-graph offset indexes,
// split over a user-chosen number of subfiles ("ADIOS allows users to control the
// number of subfiles"). Plus the comparison backend the paper measures
// against: one object file per graph.
//
// Layout of a container directory (little-endian, format version 1):
//   meta.idx   "HGPK" u32 version, i64 G, N, E, i32 F0, Fe, n_sub, reserved,
//              i64 node_offset[G+1], i64 edge_offset[G+1], i64 sub_graph[n_sub+1],
//              u32 CRC-32C of everything before it
//   data.<k>   "HGPD" u32 version, i64 g0, g1, n0, n1, e0, e1 (global ranges of
//              subfile k), then blocks:
//              x [n1-n0][F0] f32 | src [e1-e0] i32 | dst [e1-e0] i32 (graph-local) |
//              edge_attr [e1-e0][Fe] f32 | y [g1-g0] f32 (u32 CRC-32C after each block)
// Subfile k holds the contiguous graph range [sub_graph[k], sub_graph[k+1]).
// The reader reads every subfile's blocks straight into the final global arrays
// (one thread per subfile) and validates the result like hg_store_create.
#include <errno.h>
#include <sys/stat.h>
#include <sys/types.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "hgnn.h"
#include "internal.h"

namespace hg {

// CRC-32C (Castagnoli) with the SSE4.2 instruction, 8 bytes per step (container files and
// checkpoints)
uint32_t crc32c(const void *data, size_t n, uint32_t crc) {
  const uint8_t *p = (const uint8_t *)data;
  uint64_t c = ~crc;
  while (n >= 8) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    c = __builtin_ia32_crc32di(c, v);
    p += 8;
    n -= 8;
  }
  uint32_t c32 = (uint32_t)c;
  while (n--) c32 = __builtin_ia32_crc32qi(c32, *p++);
  return ~c32;
}

namespace {

constexpr uint32_t kVersion = 1;

uint32_t crc32(const void *data, size_t n, uint32_t crc = 0) { return crc32c(data, n, crc); }

struct File {
  FILE *f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

bool write_block(FILE *f, const void *p, size_t n, bool with_crc = true) {
  if (n && fwrite(p, 1, n, f) != n) return false;
  if (!with_crc) return true;
  const uint32_t c = crc32(p, n);
  return fwrite(&c, 4, 1, f) == 1;
}

bool read_block(FILE *f, void *p, size_t n) {
  if (n && fread(p, 1, n, f) != n) return false;
  uint32_t c = 0;
  if (fread(&c, 4, 1, f) != 1) return false;
  return c == crc32(p, n);
}

hg_status make_dir(const char *dir) {
  if (mkdir(dir, 0755) != 0 && errno != EEXIST) return fail(HG_E_IO, "cannot create %s: %s", dir, strerror(errno));
  return HG_OK;
}

int threads_for(int32_t t, int n) {
  int h = t > 0 ? t : (int)std::max(1u, std::thread::hardware_concurrency());
  return std::max(1, std::min(h, n));
}

// run fn(i) for i in [0, n) on up to `threads` threads; first non-OK status wins
template <class F>
hg_status run_parallel(int n, int threads, F fn) {
  std::vector<hg_status> st(n, HG_OK);
  std::vector<std::string> msg(n);
  std::vector<std::thread> th;
  const int nt = threads_for(threads, n);
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int i = t; i < n; i += nt) {
        st[i] = fn(i);
        if (st[i] != HG_OK) msg[i] = hg_last_error();
      }
    });
  for (auto &x : th) x.join();
  for (int i = 0; i < n; ++i)
    if (st[i] != HG_OK) return fail(st[i], "%s", msg[i].c_str());
  return HG_OK;
}

struct MetaHead {
  char magic[4];
  uint32_t version;
  int64_t G, N, E;
  int32_t F0, Fe, n_sub, reserved;
};
struct DataHead {
  char magic[4];
  uint32_t version;
  int64_t g0, g1, n0, n1, e0, e1;
};

hg_status adopt(hg_store *s, int32_t threads, hg_store **out) {
  s->no = s->own_no.data();
  s->eo = s->own_eo.data();
  s->x = s->own_x.data();
  s->ea = s->own_ea.data();
  s->y = s->own_y.data();
  s->src = s->own_ei.data();
  s->dst = s->own_ei.data() + s->E;
  const hg_status st = store_finish(s, threads);
  if (st != HG_OK) {
    delete s;
    return st;
  }
  *out = s;
  return HG_OK;
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

hg_status hg_container_write(const hg_store *s, const char *dir, int32_t n_subfiles, int32_t threads) {
  if (!s || !dir) return fail(HG_E_INVALID, "null argument");
  if (n_subfiles < 1 || n_subfiles > s->G) return fail(HG_E_INVALID, "n_subfiles must be in [1, #graphs]");
  hg_status st = make_dir(dir);
  if (st) return st;
  const std::string base(dir);
  std::vector<int64_t> sub(n_subfiles + 1);
  for (int k = 0; k <= n_subfiles; ++k) sub[k] = s->G * k / n_subfiles;
  st = run_parallel(n_subfiles, threads, [&](int k) -> hg_status {
    const std::string path = base + "/data." + std::to_string(k);
    File f;
    if (!(f.f = fopen(path.c_str(), "wb"))) return fail(HG_E_IO, "cannot write %s", path.c_str());
    const int64_t g0 = sub[k], g1 = sub[k + 1];
    DataHead h{{'H', 'G', 'P', 'D'}, kVersion, g0, g1, s->no[g0], s->no[g1], s->eo[g0], s->eo[g1]};
    const int64_t n = h.n1 - h.n0, e = h.e1 - h.e0;
    bool ok = write_block(f.f, &h, sizeof(h), false) &&
              write_block(f.f, s->x + h.n0 * s->F0, sizeof(float) * n * s->F0) &&
              write_block(f.f, s->src + h.e0, sizeof(int32_t) * e) && write_block(f.f, s->dst + h.e0, sizeof(int32_t) * e) &&
              write_block(f.f, s->ea + h.e0 * s->Fe, sizeof(float) * e * s->Fe) &&
              write_block(f.f, s->y + g0, sizeof(float) * (g1 - g0));
    if (!ok) return fail(HG_E_IO, "short write to %s", path.c_str());
    return HG_OK;
  });
  if (st) return st;
  // the index last: a container is readable only once every subfile is complete
  const std::string mpath = base + "/meta.idx";
  File f;
  if (!(f.f = fopen(mpath.c_str(), "wb"))) return fail(HG_E_IO, "cannot write %s", mpath.c_str());
  MetaHead m{{'H', 'G', 'P', 'K'}, kVersion, s->G, s->N, s->E, s->F0, s->Fe, n_subfiles, 0};
  uint32_t c = crc32(&m, sizeof(m));
  c = crc32(s->no, sizeof(int64_t) * (s->G + 1), c);
  c = crc32(s->eo, sizeof(int64_t) * (s->G + 1), c);
  c = crc32(sub.data(), sizeof(int64_t) * sub.size(), c);
  const bool ok = write_block(f.f, &m, sizeof(m), false) &&
                  write_block(f.f, s->no, sizeof(int64_t) * (s->G + 1), false) &&
                  write_block(f.f, s->eo, sizeof(int64_t) * (s->G + 1), false) &&
                  write_block(f.f, sub.data(), sizeof(int64_t) * sub.size(), false) && fwrite(&c, 4, 1, f.f) == 1;
  if (!ok) return fail(HG_E_IO, "short write to %s", mpath.c_str());
  return HG_OK;
}

hg_status hg_container_info(const char *dir, int64_t *graphs, int64_t *nodes, int64_t *edges, int32_t *subfiles) {
  if (!dir) return fail(HG_E_INVALID, "null argument");
  const std::string mpath = std::string(dir) + "/meta.idx";
  File f;
  if (!(f.f = fopen(mpath.c_str(), "rb"))) return fail(HG_E_IO, "cannot open %s", mpath.c_str());
  MetaHead m;
  if (fread(&m, sizeof(m), 1, f.f) != 1 || std::memcmp(m.magic, "HGPK", 4) != 0)
    return fail(HG_E_IO, "%s: bad magic", mpath.c_str());
  if (m.version != kVersion) return fail(HG_E_IO, "%s: unsupported version %u", mpath.c_str(), m.version);
  if (graphs) *graphs = m.G;
  if (nodes) *nodes = m.N;
  if (edges) *edges = m.E;
  if (subfiles) *subfiles = m.n_sub;
  return HG_OK;
}

hg_status hg_container_open(const char *dir, int32_t threads, hg_store **out) {
  if (!dir || !out) return fail(HG_E_INVALID, "null argument");
  *out = nullptr;
  const std::string base(dir), mpath = base + "/meta.idx";
  File f;
  if (!(f.f = fopen(mpath.c_str(), "rb"))) return fail(HG_E_IO, "cannot open %s", mpath.c_str());
  MetaHead m;
  if (fread(&m, sizeof(m), 1, f.f) != 1 || std::memcmp(m.magic, "HGPK", 4) != 0)
    return fail(HG_E_IO, "%s: bad magic", mpath.c_str());
  if (m.version != kVersion) return fail(HG_E_IO, "%s: unsupported version %u", mpath.c_str(), m.version);
  if (m.G < 1 || m.N < 1 || m.E < 0 || m.F0 < 1 || m.Fe < 1 || m.Fe > 8 || m.n_sub < 1 || m.n_sub > m.G)
    return fail(HG_E_IO, "%s: corrupt header", mpath.c_str());
  {  // the index must fit its file, and the data its subfiles' total size, before anything is allocated
    std::error_code ec;
    const uint64_t isz = std::filesystem::file_size(mpath, ec);
    const uint64_t need = sizeof(m) + 16ull * ((uint64_t)m.G + 1) + 8ull * ((uint64_t)m.n_sub + 1) + 4;
    if (ec || isz != need) return fail(HG_E_IO, "%s: index size %llu != %llu (corrupt header)", mpath.c_str(),
                                       (unsigned long long)isz, (unsigned long long)need);
    uint64_t dsz = 0;
    for (int32_t k = 0; k < m.n_sub; ++k) {
      const uint64_t z = std::filesystem::file_size(base + "/data." + std::to_string(k), ec);
      if (ec) return fail(HG_E_IO, "missing subfile %s/data.%d (MissingSubfile)", dir, k);
      dsz += z;
    }
    const long double bytes = 4.0L * ((long double)m.N * m.F0 + (long double)m.E * (2 + m.Fe) + m.G);
    if (bytes > (long double)dsz) return fail(HG_E_IO, "%s: header counts exceed the subfiles' size", mpath.c_str());
  }
  hg_store *s = nullptr;
  try {
    s = new hg_store();
  s->G = m.G; s->N = m.N; s->E = m.E; s->F0 = m.F0; s->Fe = m.Fe;
  s->own_no.resize(m.G + 1);
  s->own_eo.resize(m.G + 1);
  std::vector<int64_t> sub(m.n_sub + 1);
  uint32_t c = crc32(&m, sizeof(m)), stored = 0;
  bool ok = fread(s->own_no.data(), sizeof(int64_t), m.G + 1, f.f) == (size_t)(m.G + 1) &&
            fread(s->own_eo.data(), sizeof(int64_t), m.G + 1, f.f) == (size_t)(m.G + 1) &&
            fread(sub.data(), sizeof(int64_t), sub.size(), f.f) == sub.size() && fread(&stored, 4, 1, f.f) == 1;
  if (ok) {
    c = crc32(s->own_no.data(), sizeof(int64_t) * (m.G + 1), c);
    c = crc32(s->own_eo.data(), sizeof(int64_t) * (m.G + 1), c);
    c = crc32(sub.data(), sizeof(int64_t) * sub.size(), c);
    ok = c == stored && s->own_no[0] == 0 && s->own_eo[0] == 0 && s->own_no[m.G] == m.N && s->own_eo[m.G] == m.E &&
         sub[0] == 0 && sub[m.n_sub] == m.G;
    // every subfile range and every offset selects memory inside the arrays (they become fread
    // destinations below): sub strictly increasing in [0, G], offsets non-decreasing in [0, N|E]
    for (int32_t k = 0; ok && k < m.n_sub; ++k) ok = sub[k] < sub[k + 1] && sub[k + 1] <= m.G;
    for (int64_t g = 0; ok && g < m.G; ++g)
      ok = s->own_no[g] <= s->own_no[g + 1] && s->own_no[g + 1] <= m.N && s->own_eo[g] <= s->own_eo[g + 1] &&
           s->own_eo[g + 1] <= m.E;
  }
  if (!ok) {
    delete s;
    return fail(HG_E_IO, "%s: corrupt index (CorruptIndex)", mpath.c_str());
  }
  s->own_x.resize((size_t)m.N * m.F0);
  s->own_ea.resize((size_t)m.E * m.Fe);
  s->own_y.resize(m.G);
  s->own_ei.resize((size_t)2 * m.E);
  hg_status st = run_parallel(m.n_sub, threads, [&](int k) -> hg_status {
    const std::string path = base + "/data." + std::to_string(k);
    File df;
    if (!(df.f = fopen(path.c_str(), "rb"))) return fail(HG_E_IO, "missing subfile %s (MissingSubfile)", path.c_str());
    DataHead h;
    const int64_t g0 = sub[k], g1 = sub[k + 1];
    if (fread(&h, sizeof(h), 1, df.f) != 1 || std::memcmp(h.magic, "HGPD", 4) != 0 || h.version != kVersion ||
        h.g0 != g0 || h.g1 != g1 || h.n0 != s->own_no[g0] || h.n1 != s->own_no[g1] || h.e0 != s->own_eo[g0] ||
        h.e1 != s->own_eo[g1])
      return fail(HG_E_IO, "%s: header does not match the index", path.c_str());
    const int64_t n = h.n1 - h.n0, e = h.e1 - h.e0;
    const bool good = read_block(df.f, s->own_x.data() + h.n0 * m.F0, sizeof(float) * n * m.F0) &&
                      read_block(df.f, s->own_ei.data() + h.e0, sizeof(int32_t) * e) &&
                      read_block(df.f, s->own_ei.data() + m.E + h.e0, sizeof(int32_t) * e) &&
                      read_block(df.f, s->own_ea.data() + h.e0 * m.Fe, sizeof(float) * e * m.Fe) &&
                      read_block(df.f, s->own_y.data() + g0, sizeof(float) * (g1 - g0));
    if (!good) return fail(HG_E_IO, "%s: truncated or checksum mismatch (CorruptIndex)", path.c_str());
    return HG_OK;
  });
  if (st) {
    delete s;
    return st;
  }
  return adopt(s, threads, out);
  } catch (const std::bad_alloc &) {
    delete s;
    return fail(HG_E_IO, "%s: header sizes exceed the host memory (corrupt header?)", mpath.c_str());
  }
}

// ---- comparison backend: one object file per graph ("g<id>.obj": header + the
// graph's arrays), the per-object loading the paper compares ADIOS against
hg_status hg_objfiles_write(const hg_store *s, const char *dir, int32_t threads) {
  if (!s || !dir) return fail(HG_E_INVALID, "null argument");
  hg_status st = make_dir(dir);
  if (st) return st;
  const std::string base(dir);
  const int nt = threads_for(threads, (int)std::min<int64_t>(s->G, 1 << 20));
  return run_parallel(nt, nt, [&](int t) -> hg_status {
    for (int64_t g = t; g < s->G; g += nt) {
      const std::string path = base + "/g" + std::to_string(g) + ".obj";
      File f;
      if (!(f.f = fopen(path.c_str(), "wb"))) return fail(HG_E_IO, "cannot write %s", path.c_str());
      const int64_t n0 = s->no[g], n = s->no[g + 1] - n0, e0 = s->eo[g], e = s->eo[g + 1] - e0;
      const int64_t hdr[4] = {0x424F4748 /* "HGOB" */, n, e, ((int64_t)s->F0 << 32) | (uint32_t)s->Fe};
      const bool ok = write_block(f.f, hdr, sizeof(hdr), false) &&
                      write_block(f.f, s->x + n0 * s->F0, sizeof(float) * n * s->F0, false) &&
                      write_block(f.f, s->src + e0, sizeof(int32_t) * e, false) &&
                      write_block(f.f, s->dst + e0, sizeof(int32_t) * e, false) &&
                      write_block(f.f, s->ea + e0 * s->Fe, sizeof(float) * e * s->Fe, false) &&
                      write_block(f.f, s->y + g, sizeof(float), false);
      if (!ok) return fail(HG_E_IO, "short write to %s", path.c_str());
    }
    return HG_OK;
  });
}

hg_status hg_objfiles_open(const char *dir, int64_t num_graphs, int32_t threads, hg_store **out) {
  if (!dir || !out) return fail(HG_E_INVALID, "null argument");
  *out = nullptr;
  if (num_graphs < 1) return fail(HG_E_EMPTY, "no graphs");
  const std::string base(dir);
  // pass 1: read every object whole (one file open + read per graph)
  std::vector<std::vector<uint8_t>> obj((size_t)num_graphs);
  const int nt = threads_for(threads, (int)std::min<int64_t>(num_graphs, 1 << 20));
  hg_status st = run_parallel(nt, nt, [&](int t) -> hg_status {
    for (int64_t g = t; g < num_graphs; g += nt) {
      const std::string path = base + "/g" + std::to_string(g) + ".obj";
      File f;
      if (!(f.f = fopen(path.c_str(), "rb"))) return fail(HG_E_IO, "missing object %s", path.c_str());
      fseek(f.f, 0, SEEK_END);
      const long sz = ftell(f.f);
      fseek(f.f, 0, SEEK_SET);
      if (sz < 32) return fail(HG_E_IO, "%s: truncated", path.c_str());
      obj[g].resize((size_t)sz);
      if (fread(obj[g].data(), 1, (size_t)sz, f.f) != (size_t)sz) return fail(HG_E_IO, "%s: short read", path.c_str());
    }
    return HG_OK;
  });
  if (st) return st;
  // pass 2: offsets, then collate into global arrays
  hg_store *s = new hg_store();
  s->G = num_graphs;
  s->own_no.assign(num_graphs + 1, 0);
  s->own_eo.assign(num_graphs + 1, 0);
  for (int64_t g = 0; g < num_graphs; ++g) {
    int64_t hdr[4];
    std::memcpy(hdr, obj[g].data(), sizeof(hdr));
    const int32_t F0 = (int32_t)(hdr[3] >> 32), Fe = (int32_t)(hdr[3] & 0xFFFFFFFF);
    if (hdr[0] != 0x424F4748 || hdr[1] < 1 || hdr[2] < 0 || F0 < 1 || Fe < 1 || Fe > 8 ||
        (g > 0 && (F0 != s->F0 || Fe != s->Fe)) ||
        obj[g].size() != 32 + sizeof(float) * (hdr[1] * F0 + hdr[2] * Fe + 1) + sizeof(int32_t) * 2 * hdr[2]) {
      delete s;
      return fail(HG_E_IO, "object %lld: corrupt", (long long)g);
    }
    s->F0 = F0;
    s->Fe = Fe;
    s->own_no[g + 1] = s->own_no[g] + hdr[1];
    s->own_eo[g + 1] = s->own_eo[g] + hdr[2];
  }
  s->N = s->own_no[num_graphs];
  s->E = s->own_eo[num_graphs];
  s->own_x.resize((size_t)s->N * s->F0);
  s->own_ea.resize((size_t)s->E * s->Fe);
  s->own_y.resize(num_graphs);
  s->own_ei.resize((size_t)2 * s->E);
  for (int64_t g = 0; g < num_graphs; ++g) {
    const uint8_t *p = obj[g].data() + 32;
    const int64_t n = s->own_no[g + 1] - s->own_no[g], e = s->own_eo[g + 1] - s->own_eo[g];
    std::memcpy(s->own_x.data() + s->own_no[g] * s->F0, p, sizeof(float) * n * s->F0);
    p += sizeof(float) * n * s->F0;
    std::memcpy(s->own_ei.data() + s->own_eo[g], p, sizeof(int32_t) * e);
    p += sizeof(int32_t) * e;
    std::memcpy(s->own_ei.data() + s->E + s->own_eo[g], p, sizeof(int32_t) * e);
    p += sizeof(int32_t) * e;
    std::memcpy(s->own_ea.data() + s->own_eo[g] * s->Fe, p, sizeof(float) * e * s->Fe);
    p += sizeof(float) * e * s->Fe;
    std::memcpy(s->own_y.data() + g, p, sizeof(float));
  }
  obj.clear();
  return adopt(s, threads, out);
}

}  // extern "C"
