// group.cpp — multi-GPU context groups in one process (SURVEY.md §8e, §8b
// "cl_create_group(devices[], SIGNAL_SHARD | COLUMN_SHARD)").
//
// Built on the single-device C-ABI only: one cl_ctx per listed device, one host
// thread per device for the duration of a call (a solve blocks its host thread
// while it paces the graph chunks, so the devices must not share one).
//
//   SIGNAL_SHARD  independent signals (clomp_solve per column, the CLI's loop
//                 cskit.cpp:543-551) split into contiguous ranges, one per
//                 device; no data-path collective; every device holds the whole
//                 dictionary.  Results land in the caller's buffers at the
//                 shard's row offset.
//   COLUMN_SHARD  one large dictionary split by atoms (cl_create_colshard): the
//                 ranks exchange candidate records / residual rows with NCCL
//                 all-gathers per outer iteration; every rank solves the whole
//                 batch, rank 0's results are returned.
//
// The same device may be listed more than once for SIGNAL_SHARD (independent
// contexts and streams on it) — that is how the single-GPU tests drive the
// group path; NCCL refuses duplicate devices, so COLUMN_SHARD needs distinct
// ones.
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/clomp_b200.h"

struct cl_group {
  int mode = CL_GROUP_SIGNAL_SHARD;
  std::vector<cl_ctx*> ctx;
  std::vector<int> devices;
  int64_t m = 0, n = 0;
  std::string err;
};

namespace {

thread_local std::string g_group_create_error;

struct Range {
  int64_t lo, hi;
};

// Contiguous signal ranges, sizes differing by at most one.
std::vector<Range> split(int64_t B, int parts) {
  std::vector<Range> r;
  const int64_t base = B / parts, extra = B % parts;
  int64_t lo = 0;
  for (int p = 0; p < parts; ++p) {
    const int64_t len = base + (p < extra ? 1 : 0);
    r.push_back({lo, lo + len});
    lo += len;
  }
  return r;
}

}  // namespace

extern "C" {

cl_group* cl_create_group(const int* devices, int ndev, const float* a, int64_t m, int64_t n,
                          int a_layout, int mode, int* status) {
  auto bail = [&](int code, const std::string& msg) -> cl_group* {
    g_group_create_error = msg;
    if (status) *status = code;
    return nullptr;
  };
  if (!devices || ndev < 1) return bail(CL_ERR_CONFIG, "cl_create_group: no devices");
  if (mode != CL_GROUP_SIGNAL_SHARD && mode != CL_GROUP_COLUMN_SHARD)
    return bail(CL_ERR_CONFIG, "cl_create_group: unknown mode");
  if (mode == CL_GROUP_COLUMN_SHARD)
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < i; ++j)
        if (devices[i] == devices[j])
          return bail(CL_ERR_CONFIG,
                      "cl_create_group: column sharding needs distinct devices (one NCCL rank each)");
  auto* g = new cl_group();
  g->mode = mode;
  g->m = m;
  g->n = n;
  g->devices.assign(devices, devices + ndev);
  g->ctx.assign((size_t)ndev, nullptr);
  std::vector<int> st((size_t)ndev, CL_OK);
  std::vector<std::string> msg((size_t)ndev);
  char nccl_id[128] = {0};
  if (mode == CL_GROUP_COLUMN_SHARD && ndev > 1 && cl_nccl_unique_id(nccl_id) != CL_OK) {
    delete g;
    return bail(CL_ERR_CUDA, "cl_create_group: NCCL is not available in this process");
  }
  // One thread per device: the dictionary uploads (and the NCCL rendezvous of
  // the column shards, which blocks until every rank arrived) run side by side.
  std::vector<std::thread> th;
  for (int r = 0; r < ndev; ++r)
    th.emplace_back([&, r] {
      int s = CL_OK;
      g->ctx[(size_t)r] = mode == CL_GROUP_COLUMN_SHARD
                              ? cl_create_colshard(devices[r], a, m, n, a_layout, r, ndev,
                                                   ndev > 1 ? nccl_id : nullptr, &s)
                              : cl_create(devices[r], a, m, n, a_layout, &s);
      st[(size_t)r] = s;
      if (!g->ctx[(size_t)r]) msg[(size_t)r] = cl_last_error(nullptr);
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < ndev; ++r)
    if (!g->ctx[(size_t)r]) {
      const int code = st[(size_t)r] ? st[(size_t)r] : CL_ERR_CUDA;
      const std::string why = "cl_create_group: device " + std::to_string(devices[r]) + ": " + msg[(size_t)r];
      cl_destroy_group(g);
      return bail(code, why);
    }
  if (status) *status = CL_OK;
  return g;
}

void cl_destroy_group(cl_group* g) {
  if (!g) return;
  for (cl_ctx* c : g->ctx)
    if (c) cl_destroy(c);
  delete g;
}

int cl_group_size(const cl_group* g) { return g ? (int)g->ctx.size() : 0; }

cl_ctx* cl_group_context(cl_group* g, int index) {
  return g && index >= 0 && index < (int)g->ctx.size() ? g->ctx[(size_t)index] : nullptr;
}

const char* cl_group_last_error(const cl_group* g) {
  return g ? g->err.c_str() : g_group_create_error.c_str();
}

int cl_group_solve_batch(cl_group* g, const float* y, int64_t batch, int y_layout,
                         const cl_config* cfg, int mode, cl_result* out) {
  if (!g) return CL_ERR_INTERNAL;
  auto fail = [&](int code, const std::string& msg) {
    g->err = msg;
    return code;
  };
  const int W = (int)g->ctx.size();
  const int64_t m = g->m, n = g->n;
  if (!y && batch > 0) return fail(CL_ERR_DIMENSION, "clomp: null y");
  if (W == 1) {  // a group of one is the plain context
    const int st = cl_solve_batch(g->ctx[0], y, batch, y_layout, cfg, mode, out);
    if (st) g->err = cl_last_error(g->ctx[0]);
    return st;
  }
  std::vector<int> st((size_t)W, CL_OK);
  std::vector<std::thread> th;
  if (g->mode == CL_GROUP_COLUMN_SHARD) {
    // Every rank needs the whole batch and joins every collective; rank 0's
    // results are the caller's (the others' are identical and dropped).
    for (int r = 0; r < W; ++r)
      th.emplace_back([&, r] {
        cl_result none{};
        st[(size_t)r] = cl_solve_batch(g->ctx[(size_t)r], y, batch, y_layout, cfg, mode,
                                       r == 0 ? out : &none);
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < W; ++r)
      if (st[(size_t)r]) return fail(st[(size_t)r], cl_last_error(g->ctx[(size_t)r]));
    return CL_OK;
  }
  // SIGNAL_SHARD
  if (mode != CL_MODE_PER_SIGNAL && batch > 1)
    return fail(CL_ERR_UNSUPPORTED,
                "cl_group_solve_batch: a joint batch couples its columns (clomp.cpp:235-273) and "
                "cannot be sharded by signal; use CL_MODE_PER_SIGNAL or a column-sharded group");
  if (batch <= 0) {  // let one context produce the reference's error
    const int s0 = cl_solve_batch(g->ctx[0], y, batch, y_layout, cfg, mode, out);
    if (s0) g->err = cl_last_error(g->ctx[0]);
    return s0;
  }
  const std::vector<Range> rg = split(batch, W);
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      const int64_t lo = rg[(size_t)r].lo, nb = rg[(size_t)r].hi - lo;
      if (nb == 0) return;
      // This shard's columns, contiguous: signal-major rows are already; the
      // reference's m x B interleaved layout is gathered into m x nb.
      const float* ys = nullptr;
      std::vector<float> gathered;
      if (y_layout == CL_LAYOUT_T) {
        ys = y + lo * m;
      } else {
        gathered.resize((size_t)(m * nb));
        for (int64_t i = 0; i < m; ++i)
          std::memcpy(&gathered[(size_t)(i * nb)], y + i * batch + lo, (size_t)nb * sizeof(float));
        ys = gathered.data();
      }
      cl_result part{};
      std::vector<double> s_part;
      std::vector<uint8_t> mask_part;
      std::vector<double> x_part;
      if (out) {
        part.cap = out->cap;
        part.support = out->support ? out->support + lo * out->cap : nullptr;
        part.coef = out->coef ? out->coef + lo * out->cap : nullptr;
        part.count = out->count ? out->count + lo : nullptr;
        part.iterations = out->iterations ? out->iterations + lo : nullptr;
        part.final_residual_norm = out->final_residual_norm ? out->final_residual_norm + lo : nullptr;
        part.converged = out->converged ? out->converged + lo : nullptr;
        part.status = out->status ? out->status + lo : nullptr;
        // dense n x B outputs interleave the signals: solve into n x nb, scatter
        if (out->s) {
          s_part.assign((size_t)(n * nb), 0.0);
          part.s = s_part.data();
        }
        if (out->mask) {
          mask_part.assign((size_t)(n * nb), 0);
          part.mask = mask_part.data();
        }
        if (out->x_hat) {
          x_part.assign((size_t)(n * nb), 0.0);
          part.x_hat = x_part.data();
        }
        part.flags = CL_RESULT_PREZEROED;
      }
      st[(size_t)r] = cl_solve_batch(g->ctx[(size_t)r], ys, nb, y_layout, cfg, mode,
                                     out ? &part : nullptr);
      if (st[(size_t)r] || !out) return;
      for (int64_t j = 0; j < n; ++j) {
        if (out->s) std::memcpy(out->s + j * batch + lo, &s_part[(size_t)(j * nb)], (size_t)nb * 8);
        if (out->mask) std::memcpy(out->mask + j * batch + lo, &mask_part[(size_t)(j * nb)], (size_t)nb);
        if (out->x_hat) std::memcpy(out->x_hat + j * batch + lo, &x_part[(size_t)(j * nb)], (size_t)nb * 8);
      }
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < W; ++r)
    if (st[(size_t)r]) return fail(st[(size_t)r], cl_last_error(g->ctx[(size_t)r]));
  return CL_OK;
}

}  // extern "C"
