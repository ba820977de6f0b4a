/*
 * molgen.c — seeded synthetic molecular-graph generator.
 *
 * INPUT GENERATOR ONLY. It holds none of the method's arithmetic: it draws
 * molecules and encodes them as the Table-1 quadruple (x, edge_index,
 * edge_attr, y) of PAPER.md:232-253 (§3.3, Table 1), with the feature
 * encoding SPEC.md:104, 121-129 (graphenc.encode_graph) fixes. Both the CPU
 * oracle (oracle/) and the CUDA product path (paper_2207_11333_b200/) read
 * its arrays; neither side's arithmetic lives here.
 *
 * Recipe:
 *   1. heavy-atom count k ~ U[kmin, kmax]
 *   2. elements drawn with C dominant (C .70, O .12, N .10, F .03, S .03,
 *      the rest of the vocabulary shares the remaining mass)
 *   3. random valence-respecting spanning forest (an atom with no free
 *      valence left anywhere, or valence 0 (noble gases), starts a new
 *      component -> isolated / disconnected nodes, PAPER/SPEC allow salts)
 *   4. Poisson(rho * k) ring closures between non-bonded atoms with free valence
 *   5. bond upgrades: double p=.15, triple p=.02, aromatic flag p=.06
 *   6. explicit hydrogens appended after the heavy atoms
 *   7. encode: x = one-hot(element) ++ [degree, formal charge, aromatic];
 *      directed edges sorted by (src,dst); edge_attr one-hot(single, double,
 *      triple, aromatic)
 *   8. y = 9.0 - 0.12 k - 0.8 (#double)/k + N(0, 0.1^2)  [eV; arbitrary]
 *
 * Randomness: every graph id g draws from its own splitmix64 stream seeded by
 * (seed, g), so any id range can be generated independently and in parallel
 * with identical results.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MG_MAX_HEAVY 64
#define MG_MAX_NODES 160
#define MG_MAX_BONDS 320
#define MG_MAX_VOCAB 64

typedef struct { const char *sym; int z; int valence; } mg_elem;

/* 31 PCQM4Mv2 elements, valences: SPEC.md:73 where given,
 * otherwise the element's common valence; noble gases 0. */
static const mg_elem k_elems[] = {
  {"H", 1, 1},  {"He", 2, 0}, {"Li", 3, 1},  {"Be", 4, 2},  {"B", 5, 3},
  {"C", 6, 4},  {"N", 7, 3},  {"O", 8, 2},   {"F", 9, 1},   {"Ne", 10, 0},
  {"Na", 11, 1},{"Mg", 12, 2},{"Al", 13, 3}, {"Si", 14, 4}, {"P", 15, 3},
  {"S", 16, 2}, {"Cl", 17, 1},{"Ar", 18, 0}, {"Ca", 20, 2}, {"Ti", 22, 4},
  {"V", 23, 3}, {"Ni", 28, 2},{"Cu", 29, 1}, {"Zn", 30, 2}, {"Ga", 31, 3},
  {"Ge", 32, 4},{"As", 33, 3},{"Se", 34, 2}, {"Br", 35, 1}, {"Kr", 36, 0},
  {"I", 53, 1},
};
#define MG_N_ELEMS ((int)(sizeof(k_elems) / sizeof(k_elems[0])))

typedef struct {
  int n_vocab;
  int vocab_z[MG_MAX_VOCAB];   /* sorted by atomic number */
  int vocab_val[MG_MAX_VOCAB];
  double cum_w[MG_MAX_VOCAB];  /* cumulative heavy-atom draw weights (H excluded) */
  int kmin, kmax, max_nodes;
  double rho;                  /* ring closures per heavy atom (Poisson mean rho*k) */
  double p_double, p_triple, p_arom, p_charge;
} mg_preset;

enum { MG_TINY = 0, MG_PCQM = 1, MG_AISD = 2 };

static int mg_find(int z) {
  for (int i = 0; i < MG_N_ELEMS; ++i) if (k_elems[i].z == z) return i;
  return -1;
}

static int mg_make_preset(int preset, mg_preset *p) {
  memset(p, 0, sizeof(*p));
  if (preset == MG_TINY || preset == MG_PCQM) {
    for (int i = 0; i < MG_N_ELEMS; ++i) {
      p->vocab_z[i] = k_elems[i].z;
      p->vocab_val[i] = k_elems[i].valence;
    }
    p->n_vocab = MG_N_ELEMS;
  } else if (preset == MG_AISD) {
    static const int z[6] = {1, 6, 7, 8, 9, 16}; /* H C N O F S */
    for (int i = 0; i < 6; ++i) {
      p->vocab_z[i] = z[i];
      p->vocab_val[i] = k_elems[mg_find(z[i])].valence;
    }
    p->n_vocab = 6;
  } else {
    return -1;
  }
  /* heavy-atom weights */
  double w[MG_MAX_VOCAB] = {0};
  int n_rest = 0;
  for (int i = 0; i < p->n_vocab; ++i) {
    int z = p->vocab_z[i];
    if (z == 1) w[i] = 0.0;
    else if (z == 6) w[i] = 0.70;
    else if (z == 8) w[i] = 0.12;
    else if (z == 7) w[i] = 0.10;
    else if (z == 9) w[i] = 0.03;
    else if (z == 16) w[i] = 0.03;
    else { w[i] = -1.0; ++n_rest; }
  }
  for (int i = 0; i < p->n_vocab; ++i) if (w[i] < 0) w[i] = 0.02 / n_rest;
  double s = 0.0;
  for (int i = 0; i < p->n_vocab; ++i) s += w[i];
  double c = 0.0;
  for (int i = 0; i < p->n_vocab; ++i) { c += w[i] / s; p->cum_w[i] = c; }
  p->cum_w[p->n_vocab - 1] = 1.0;
  p->p_double = 0.15; p->p_triple = 0.02; p->p_arom = 0.06; p->p_charge = 0.01;
  if (preset == MG_TINY) { p->kmin = 1; p->kmax = 9; p->max_nodes = 20; p->rho = 0.12; }
  if (preset == MG_PCQM) { p->kmin = 4; p->kmax = 23; p->max_nodes = 51; p->rho = 0.115; }
  if (preset == MG_AISD) { p->kmin = 12; p->kmax = 32; p->max_nodes = 100; p->rho = 0.040; }
  return 0;
}

/* ---- counter-based RNG: splitmix64 stream per (seed, graph id) ---- */
typedef struct { uint64_t s; } mg_rng;
static inline uint64_t mg_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t mg_next(mg_rng *r) { r->s += 0x9E3779B97F4A7C15ULL; return mg_mix(r->s); }
static inline double mg_unif(mg_rng *r) { return (double)(mg_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline int mg_int(mg_rng *r, int lo, int hi) { /* inclusive */
  return lo + (int)(mg_unif(r) * (double)(hi - lo + 1));
}
static int mg_poisson(mg_rng *r, double lam) {
  double L = exp(-lam), p = 1.0; int k = 0;
  do { ++k; p *= mg_unif(r); } while (p > L && k < 64);
  return k - 1;
}
static double mg_normal(mg_rng *r) {
  double u1 = mg_unif(r), u2 = mg_unif(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

typedef struct {
  int n_nodes, n_bonds;
  int elem[MG_MAX_NODES];       /* vocab index */
  int charge[MG_MAX_NODES];
  int arom[MG_MAX_NODES];
  int deg[MG_MAX_NODES];
  int ba[MG_MAX_BONDS], bb[MG_MAX_BONDS], bo[MG_MAX_BONDS]; /* order 0..3 */
  float y;
} mg_mol;

/* draw one molecule; returns 0 if it fits max_nodes, else -1 (caller redraws) */
static int mg_draw(const mg_preset *p, mg_rng *r, mg_mol *m) {
  int k = mg_int(r, p->kmin, p->kmax);
  int freev[MG_MAX_NODES];
  unsigned char adj[MG_MAX_HEAVY][MG_MAX_HEAVY];
  memset(adj, 0, sizeof(adj));
  m->n_bonds = 0;
  int h_idx = -1;
  for (int i = 0; i < p->n_vocab; ++i) if (p->vocab_z[i] == 1) h_idx = i;
  for (int a = 0; a < k; ++a) {
    double u = mg_unif(r);
    int e = 0;
    while (e < p->n_vocab - 1 && u > p->cum_w[e]) ++e;
    if (e == h_idx) e = (e + 1) % p->n_vocab;
    m->elem[a] = e; m->charge[a] = 0; m->arom[a] = 0;
    freev[a] = p->vocab_val[e];
    if (p->vocab_z[e] == 7 && mg_unif(r) < p->p_charge) { m->charge[a] = 1; freev[a] = 4; }
    if (p->vocab_z[e] == 8 && mg_unif(r) < p->p_charge) { m->charge[a] = -1; freev[a] = 1; }
  }
  /* 3. spanning forest */
  for (int a = 1; a < k; ++a) {
    if (freev[a] < 1) continue;
    int b = -1;
    for (int t = 0; t < 8 && b < 0; ++t) {
      int c = mg_int(r, 0, a - 1);
      if (freev[c] >= 1) b = c;
    }
    if (b < 0) for (int c = a - 1; c >= 0; --c) if (freev[c] >= 1) { b = c; break; }
    if (b < 0) continue; /* new component */
    m->ba[m->n_bonds] = b; m->bb[m->n_bonds] = a; m->bo[m->n_bonds] = 0; ++m->n_bonds;
    adj[a][b] = adj[b][a] = 1; --freev[a]; --freev[b];
  }
  /* 4. ring closures */
  int R = mg_poisson(r, p->rho * k);
  for (int t = 0; t < R; ++t) {
    for (int tries = 0; tries < 16; ++tries) {
      int a = mg_int(r, 0, k - 1), b = mg_int(r, 0, k - 1);
      if (a == b || adj[a][b] || freev[a] < 1 || freev[b] < 1) continue;
      m->ba[m->n_bonds] = a < b ? a : b; m->bb[m->n_bonds] = a < b ? b : a; m->bo[m->n_bonds] = 0;
      ++m->n_bonds; adj[a][b] = adj[b][a] = 1; --freev[a]; --freev[b];
      break;
    }
  }
  /* 5. bond upgrades */
  int n_double = 0;
  for (int q = 0; q < m->n_bonds; ++q) {
    int a = m->ba[q], b = m->bb[q];
    double u = mg_unif(r);
    if (u < p->p_triple) {
      if (freev[a] >= 2 && freev[b] >= 2) { m->bo[q] = 2; freev[a] -= 2; freev[b] -= 2; }
    } else if (u < p->p_triple + p->p_double) {
      if (freev[a] >= 1 && freev[b] >= 1) { m->bo[q] = 1; --freev[a]; --freev[b]; ++n_double; }
    } else if (u < p->p_triple + p->p_double + p->p_arom) {
      m->bo[q] = 3; m->arom[a] = 1; m->arom[b] = 1;
    }
  }
  /* 6. explicit hydrogens */
  int n = k;
  for (int a = 0; a < k; ++a) {
    for (int h = 0; h < freev[a]; ++h) {
      if (n >= MG_MAX_NODES || m->n_bonds >= MG_MAX_BONDS) return -1;
      m->elem[n] = h_idx; m->charge[n] = 0; m->arom[n] = 0;
      m->ba[m->n_bonds] = a; m->bb[m->n_bonds] = n; m->bo[m->n_bonds] = 0; ++m->n_bonds;
      ++n;
    }
  }
  m->n_nodes = n;
  if (n > p->max_nodes) return -1;
  for (int a = 0; a < n; ++a) m->deg[a] = 0;
  for (int q = 0; q < m->n_bonds; ++q) { ++m->deg[m->ba[q]]; ++m->deg[m->bb[q]]; }
  double y = 9.0 - 0.12 * k - 0.8 * (double)n_double / (double)k + 0.1 * mg_normal(r);
  m->y = (float)y;
  return 0;
}

static void mg_seed(mg_rng *r, uint64_t seed, int64_t g) {
  r->s = mg_mix(seed ^ ((uint64_t)g * 0xD1B54A32D192ED03ULL) ^ 0x6A09E667F3BCC909ULL);
}

static void mg_gen(const mg_preset *p, uint64_t seed, int64_t g, mg_mol *m) {
  mg_rng r; mg_seed(&r, seed, g);
  while (mg_draw(p, &r, m) != 0) { /* redraw from the same stream */ }
}

typedef struct { int src, dst, order; } mg_edge;
static int mg_edge_cmp(const void *a, const void *b) {
  const mg_edge *x = (const mg_edge *)a, *y = (const mg_edge *)b;
  if (x->src != y->src) return x->src - y->src;
  return x->dst - y->dst;
}

/* ------------------------------- public API ------------------------------ */

int molgen_preset_info(int preset, int32_t *n_vocab, int32_t *f_node, int32_t *f_edge,
                       int32_t *max_nodes, int32_t *vocab_z) {
  mg_preset p;
  if (mg_make_preset(preset, &p)) return -1;
  *n_vocab = p.n_vocab; *f_node = p.n_vocab + 3; *f_edge = 4; *max_nodes = p.max_nodes;
  if (vocab_z) for (int i = 0; i < p.n_vocab; ++i) vocab_z[i] = p.vocab_z[i];
  return 0;
}

typedef struct {
  const mg_preset *p; uint64_t seed; int64_t g0, n; int tid, nthreads;
  int32_t *nodes, *edges;                       /* count mode */
  const int64_t *node_offset, *edge_offset;     /* fill mode */
  int64_t e_total; float *x; int32_t *ei; float *ea; float *y;
} mg_job;

static void *mg_count_worker(void *arg) {
  mg_job *j = (mg_job *)arg;
  mg_mol m;
  for (int64_t i = j->tid; i < j->n; i += j->nthreads) {
    mg_gen(j->p, j->seed, j->g0 + i, &m);
    j->nodes[i] = m.n_nodes; j->edges[i] = 2 * m.n_bonds;
  }
  return NULL;
}

static void *mg_fill_worker(void *arg) {
  mg_job *j = (mg_job *)arg;
  const int F = j->p->n_vocab + 3;
  mg_mol m;
  mg_edge es[2 * MG_MAX_BONDS];
  for (int64_t i = j->tid; i < j->n; i += j->nthreads) {
    mg_gen(j->p, j->seed, j->g0 + i, &m);
    int64_t n0 = j->node_offset[i] - j->node_offset[0];
    int64_t e0 = j->edge_offset[i] - j->edge_offset[0];
    float *xr = j->x + n0 * F;
    memset(xr, 0, sizeof(float) * (size_t)m.n_nodes * F);
    for (int a = 0; a < m.n_nodes; ++a) {
      xr[a * F + m.elem[a]] = 1.0f;
      xr[a * F + j->p->n_vocab + 0] = (float)m.deg[a];
      xr[a * F + j->p->n_vocab + 1] = (float)m.charge[a];
      xr[a * F + j->p->n_vocab + 2] = (float)m.arom[a];
    }
    int ne = 0;
    for (int q = 0; q < m.n_bonds; ++q) {
      es[ne].src = m.ba[q]; es[ne].dst = m.bb[q]; es[ne].order = m.bo[q]; ++ne;
      es[ne].src = m.bb[q]; es[ne].dst = m.ba[q]; es[ne].order = m.bo[q]; ++ne;
    }
    qsort(es, ne, sizeof(mg_edge), mg_edge_cmp);
    for (int q = 0; q < ne; ++q) {
      j->ei[e0 + q] = es[q].src;
      j->ei[j->e_total + e0 + q] = es[q].dst;
      float *ar = j->ea + (e0 + q) * 4;
      ar[0] = ar[1] = ar[2] = ar[3] = 0.0f;
      ar[es[q].order] = 1.0f;
    }
    j->y[i] = m.y;
  }
  return NULL;
}

static int mg_run(mg_job *proto, void *(*fn)(void *), int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  mg_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = *proto; jobs[t].tid = t; jobs[t].nthreads = threads;
    if (pthread_create(&th[t], NULL, fn, &jobs[t])) return -2;
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* per-graph node and directed-edge counts for graphs [g0, g0+n) */
int molgen_count(int preset, uint64_t seed, int64_t g0, int64_t n,
                 int32_t *nodes, int32_t *edges, int threads) {
  mg_preset p;
  if (mg_make_preset(preset, &p)) return -1;
  mg_job j; memset(&j, 0, sizeof(j));
  j.p = &p; j.seed = seed; j.g0 = g0; j.n = n; j.nodes = nodes; j.edges = edges;
  return mg_run(&j, mg_count_worker, threads);
}

/* fill Table-1 arrays; offsets are the [n+1] prefix sums of molgen_count;
 * edge_index is [2][e_total] (row 0 src, row 1 dst), graph-local ids. */
int molgen_fill(int preset, uint64_t seed, int64_t g0, int64_t n,
                const int64_t *node_offset, const int64_t *edge_offset, int64_t e_total,
                float *x, int32_t *edge_index, float *edge_attr, float *y, int threads) {
  mg_preset p;
  if (mg_make_preset(preset, &p)) return -1;
  mg_job j; memset(&j, 0, sizeof(j));
  j.p = &p; j.seed = seed; j.g0 = g0; j.n = n;
  j.node_offset = node_offset; j.edge_offset = edge_offset; j.e_total = e_total;
  j.x = x; j.ei = edge_index; j.ea = edge_attr; j.y = y;
  return mg_run(&j, mg_fill_worker, threads);
}
