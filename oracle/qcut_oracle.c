/*
 * qcut_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's per-slice hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CPU oracle.
 * The product (paper_2010_14962_b200/) never links or calls this file.
 *
 * It restates, over a leg dimension D in {4 (density view, the reference's
 * own), 2 (ket view, SURVEY.md §8 conventions)}:
 *   sum_range        proj/core/src/executor.cpp:45-68   (ascending acc +=)
 *   assignment digits proj/core/src/cutting.cpp:41-52   (MSB = first cut edge)
 *   apply_cut        proj/core/src/cutting.cpp:67-129   (+ slice_legs tensor.cpp:79-105,
 *                                                        slice_leg_map tensor.cpp:64-77)
 *   execute_plan     proj/core/src/contraction.cpp:288-319
 *   contract_pair    proj/core/src/contraction.cpp:71-116 (+ free_legs :58-67,
 *                                                        permute_legs tensor.cpp:30-62)
 * with the same loop orders (i-s-j MAC with the zero skip on e[i,s]) so that
 * density-view results are bit-identical to the reference except for the
 * order leftover rank-0 tensors are multiplied in (the reference iterates an
 * unordered_map; we use ascending vertex id).
 *
 * Input is a flattened payload (see oracle/oracle.py): vertices with rank and
 * D^rank complex values, edges (id,u,leg_u,v,leg_v), sorted cut edge ids, plan
 * steps (a, b, shared legs) and plan scalars.
 *
 * Parity status: pinned against the compiled reference (oracle/_ref/qcut_refgen)
 * on the committed golden fixtures, see tests/test_oracle_golden.py.
 */
#include <errno.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cxd;

static inline cxd cmul(cxd a, cxd b) {
  cxd r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

typedef struct {
  int rank;
  size_t size;
  cxd* data;
} tensor_t;

typedef struct {
  int D;          /* leg dimension: 4 density, 2 ket */
  int nv;         /* vertices */
  const int* vid; /* vertex ids (ascending) */
  const int* vrank;
  const int64_t* voff; /* offset (in complex elements) of each vertex's data */
  const double* vdata; /* interleaved re,im */
  int ne;
  const int* e_id;
  const int* e_u;
  const int* e_lu;
  const int* e_v;
  const int* e_lv;
  int M;
  const int* cut;
  int nsteps;
  const int* st_a;
  const int* st_b;
  const int* st_k;     /* shared legs per step */
  const int* st_off;   /* offset into st_la / st_lb */
  const int* st_la;
  const int* st_lb;
  int nscal;
  const int* scal;
} qo_net;

static size_t ipow(int D, int r) {
  size_t s = 1;
  for (int i = 0; i < r; ++i) s *= (size_t)D;
  return s;
}

static __thread char g_err[512];
const char* qo_last_error(void) { return g_err; }

/* permute_legs (tensor.cpp:30-62): perm[i] = source leg of output leg i. */
static tensor_t permute(const tensor_t* t, const int* perm, int D) {
  tensor_t o;
  o.rank = t->rank;
  o.size = t->size;
  o.data = (cxd*)malloc(sizeof(cxd) * (o.size ? o.size : 1));
  if (t->rank <= 1) {
    memcpy(o.data, t->data, sizeof(cxd) * t->size);
    return o;
  }
  size_t in_stride[64];
  int digit[64];
  for (int p = 0; p < t->rank; ++p) {
    in_stride[p] = ipow(D, t->rank - 1 - perm[p]);
    digit[p] = 0;
  }
  size_t in_idx = 0;
  for (size_t out_idx = 0; out_idx < o.size; ++out_idx) {
    o.data[out_idx] = t->data[in_idx];
    for (int p = t->rank - 1; p >= 0; --p) {
      in_idx += in_stride[p];
      if (++digit[p] < D) break;
      digit[p] = 0;
      in_idx -= (size_t)D * in_stride[p];
    }
  }
  return o;
}

/* contract_pair (contraction.cpp:71-116). */
static int contract(const tensor_t* e, const int* le, const tensor_t* f, const int* lf,
                    int k, int D, tensor_t* g) {
  int fe[64], ff[64], nfe = 0, nff = 0;
  char se[64] = {0}, sf[64] = {0};
  for (int i = 0; i < k; ++i) {
    if (le[i] < 0 || le[i] >= e->rank || se[le[i]]) return -1;
    if (lf[i] < 0 || lf[i] >= f->rank || sf[lf[i]]) return -1;
    se[le[i]] = 1;
    sf[lf[i]] = 1;
  }
  for (int l = 0; l < e->rank; ++l)
    if (!se[l]) fe[nfe++] = l;
  for (int l = 0; l < f->rank; ++l)
    if (!sf[l]) ff[nff++] = l;
  int pe_perm[64], pf_perm[64];
  for (int i = 0; i < nfe; ++i) pe_perm[i] = fe[i];
  for (int i = 0; i < k; ++i) pe_perm[nfe + i] = le[i];
  for (int i = 0; i < k; ++i) pf_perm[i] = lf[i];
  for (int i = 0; i < nff; ++i) pf_perm[k + i] = ff[i];
  tensor_t pe = permute(e, pe_perm, D);
  tensor_t pf = permute(f, pf_perm, D);
  size_t m = ipow(D, nfe), kk = ipow(D, k), n = ipow(D, nff);
  g->rank = nfe + nff;
  g->size = m * n;
  g->data = (cxd*)calloc(g->size ? g->size : 1, sizeof(cxd));
  for (size_t i = 0; i < m; ++i) {
    const cxd* a_row = pe.data + i * kk;
    cxd* g_row = g->data + i * n;
    for (size_t s = 0; s < kk; ++s) {
      cxd a = a_row[s];
      if (a.re == 0.0 && a.im == 0.0) continue;
      const cxd* b_row = pf.data + s * n;
      for (size_t j = 0; j < n; ++j) {
        cxd p = cmul(a, b_row[j]);
        g_row[j].re += p.re;
        g_row[j].im += p.im;
      }
    }
  }
  free(pe.data);
  free(pf.data);
  return 0;
}

/* slice_legs (tensor.cpp:79-105) for a vertex with `nf` (leg, digit) fixes. */
static tensor_t slice_tensor(const tensor_t* t, const int* fleg, const int* fdig, int nf, int D) {
  char fixed[64] = {0};
  size_t base = 0;
  for (int i = 0; i < nf; ++i) {
    fixed[fleg[i]] = 1;
    base += (size_t)fdig[i] * ipow(D, t->rank - 1 - fleg[i]);
  }
  size_t kept_stride[64];
  int nk = 0;
  for (int l = 0; l < t->rank; ++l)
    if (!fixed[l]) kept_stride[nk++] = ipow(D, t->rank - 1 - l);
  tensor_t o;
  o.rank = nk;
  o.size = ipow(D, nk);
  o.data = (cxd*)malloc(sizeof(cxd) * o.size);
  int digit[64] = {0};
  size_t in_idx = base;
  for (size_t out_idx = 0; out_idx < o.size; ++out_idx) {
    o.data[out_idx] = t->data[in_idx];
    for (int p = nk - 1; p >= 0; --p) {
      in_idx += kept_stride[p];
      if (++digit[p] < D) break;
      digit[p] = 0;
      in_idx -= (size_t)D * kept_stride[p];
    }
  }
  return o;
}

static int vindex(const qo_net* n, int id) {
  int lo = 0, hi = n->nv - 1;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (n->vid[mid] == id) return mid;
    if (n->vid[mid] < id) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

/* One slice: apply_cut (cutting.cpp:67-129) then execute_plan (contraction.cpp:288-319).
 * Plan legs are already in the cut network's coordinates (the plan was made on
 * apply_cut(tn, cut, 0...0), executor.cpp:33-43), so only tensor data needs
 * slicing here. */
static int run_slice(const qo_net* n, uint64_t idx, cxd* out) {
  const int D = n->D;
  const int bits = D == 4 ? 2 : 1;
  tensor_t* live = (tensor_t*)calloc((size_t)n->nv, sizeof(tensor_t));
  char* alive = (char*)calloc((size_t)n->nv, 1);
  /* per-vertex fixes from the cut */
  int* nfix = (int*)calloc((size_t)n->nv, sizeof(int));
  int* fleg = (int*)malloc(sizeof(int) * (size_t)n->nv * 8);
  int* fdig = (int*)malloc(sizeof(int) * (size_t)n->nv * 8);
  int rc = 0;
  for (int i = 0; i < n->M; ++i) {
    int digit = (int)((idx >> (bits * (n->M - 1 - i))) & (uint64_t)(D - 1));
    int ei = -1;
    for (int j = 0; j < n->ne; ++j)
      if (n->e_id[j] == n->cut[i]) ei = j;
    if (ei < 0) {
      snprintf(g_err, sizeof g_err, "cut references unknown edge %d", n->cut[i]);
      rc = -1;
      goto done;
    }
    int ends[2][2] = {{n->e_u[ei], n->e_lu[ei]}, {n->e_v[ei], n->e_lv[ei]}};
    for (int s = 0; s < 2; ++s) {
      int vi = vindex(n, ends[s][0]);
      int c = nfix[vi]++;
      fleg[vi * 8 + c] = ends[s][1];
      fdig[vi * 8 + c] = digit;
    }
  }
  for (int vi = 0; vi < n->nv; ++vi) {
    tensor_t t;
    t.rank = n->vrank[vi];
    t.size = ipow(D, t.rank);
    t.data = (cxd*)(n->vdata + 2 * n->voff[vi]);
    if (nfix[vi]) {
      /* fixes sorted by leg (cutting.cpp:115) — order does not change the result */
      live[vi] = slice_tensor(&t, fleg + vi * 8, fdig + vi * 8, nfix[vi], D);
    } else {
      live[vi].rank = t.rank;
      live[vi].size = t.size;
      live[vi].data = (cxd*)malloc(sizeof(cxd) * t.size);
      memcpy(live[vi].data, t.data, sizeof(cxd) * t.size);
    }
    alive[vi] = 1;
  }
  cxd acc = {1.0, 0.0};
  for (int s = 0; s < n->nsteps; ++s) {
    int ia = vindex(n, n->st_a[s]), ib = vindex(n, n->st_b[s]);
    if (ia < 0 || ib < 0 || !alive[ia] || !alive[ib]) {
      snprintf(g_err, sizeof g_err, "plan references a missing vertex");
      rc = -1;
      goto done;
    }
    tensor_t g;
    if (contract(&live[ia], n->st_la + n->st_off[s], &live[ib], n->st_lb + n->st_off[s],
                 n->st_k[s], D, &g)) {
      snprintf(g_err, sizeof g_err, "bad leg list at step %d", s);
      rc = -1;
      goto done;
    }
    free(live[ib].data);
    live[ib].data = NULL;
    alive[ib] = 0;
    free(live[ia].data);
    if (g.rank == 0) {
      acc = cmul(acc, g.data[0]);
      free(g.data);
      live[ia].data = NULL;
      alive[ia] = 0;
    } else {
      live[ia] = g;
    }
  }
  for (int vi = 0; vi < n->nv; ++vi) {
    if (!alive[vi]) continue;
    if (live[vi].rank != 0) {
      snprintf(g_err, sizeof g_err, "plan does not reduce vertex %d to a scalar", n->vid[vi]);
      rc = -1;
      goto done;
    }
    acc = cmul(acc, live[vi].data[0]);
  }
  *out = acc;
done:
  for (int vi = 0; vi < n->nv; ++vi) free(live[vi].data);
  free(live);
  free(alive);
  free(nfix);
  free(fleg);
  free(fdig);
  return rc;
}

/* sum_range (executor.cpp:45-68): ascending slice order, acc +=. If `per_slice`
 * is non-NULL it receives hi-lo values (interleaved re,im). */
int qo_sum_range(const qo_net* n, uint64_t lo, uint64_t hi, double* out2, double* per_slice) {
  uint64_t total = (uint64_t)1 << ((n->D == 4 ? 2 : 1) * n->M);
  if (lo > hi || hi > total) {
    snprintf(g_err, sizeof g_err, "range [%llu,%llu) outside [0,%llu)",
             (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)total);
    return EINVAL;
  }
  cxd acc = {0.0, 0.0};
  for (uint64_t idx = lo; idx < hi; ++idx) {
    cxd v;
    if (run_slice(n, idx, &v)) return EINVAL;
    if (per_slice) {
      per_slice[2 * (idx - lo)] = v.re;
      per_slice[2 * (idx - lo) + 1] = v.im;
    }
    acc.re += v.re;
    acc.im += v.im;
  }
  out2[0] = acc.re;
  out2[1] = acc.im;
  return 0;
}

typedef struct {
  const qo_net* n;
  uint64_t lo, hi;
  double v[2];
  int rc;
} qo_job;

static void* qo_worker(void* p) {
  qo_job* j = (qo_job*)p;
  j->rc = qo_sum_range(j->n, j->lo, j->hi, j->v, NULL);
  return NULL;
}

/* run_pool (executor.cpp:113-176) default grid: ceil(count/workers) contiguous
 * batches, partials folded in ascending lo order (aggregate, :78-111). */
int qo_sum_range_pool(const qo_net* n, uint64_t lo, uint64_t hi, int workers, double* out2) {
  if (workers < 1) workers = 1;
  if (lo > hi) return EINVAL;
  uint64_t count = hi - lo;
  uint64_t batch = (count + (uint64_t)workers - 1) / (uint64_t)workers;
  if (batch == 0) batch = 1;
  qo_job* jobs = (qo_job*)calloc((size_t)workers, sizeof(qo_job));
  pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
  for (int w = 0; w < workers; ++w) {
    uint64_t a = lo + (uint64_t)w * batch;
    if (a > hi) a = hi;
    uint64_t b = a + batch > hi ? hi : a + batch;
    jobs[w].n = n;
    jobs[w].lo = a;
    jobs[w].hi = b;
    pthread_create(&th[w], NULL, qo_worker, &jobs[w]);
  }
  int rc = 0;
  double acc[2] = {0.0, 0.0};
  for (int w = 0; w < workers; ++w) {
    pthread_join(th[w], NULL);
    if (jobs[w].rc) rc = jobs[w].rc;
  }
  for (int w = 0; w < workers; ++w) {
    acc[0] += jobs[w].v[0];
    acc[1] += jobs[w].v[1];
  }
  out2[0] = acc[0];
  out2[1] = acc[1];
  free(jobs);
  free(th);
  return rc;
}

/* Standalone contract_pair for known-answer tests (test_contraction.cpp:46-106). */
int qo_contract_pair(int D, int rank_e, const double* e, const int* le, int rank_f,
                     const double* f, const int* lf, int k, double* out) {
  tensor_t te = {rank_e, ipow(D, rank_e), (cxd*)e};
  tensor_t tf = {rank_f, ipow(D, rank_f), (cxd*)f};
  tensor_t g;
  if (contract(&te, le, &tf, lf, k, D, &g)) return EINVAL;
  memcpy(out, g.data, sizeof(cxd) * g.size);
  free(g.data);
  return 0;
}
