// patchmg_gpu.hpp -- header-only C++ mirror of the reference's Backend seam
// over libpmg_cuda's C ABI (include/pmg_cuda.h).
//
// GpuBackend satisfies the Backend concept consumed by mg_cycle_generic /
// mg_precondition / pcg_generic (/root/reference/proj/include/patchmg/
// multigrid.hpp:120-189), with the same method names, argument meaning and
// error behaviour as SerialBackend (multigrid.hpp:80-114) and ParallelBackend
// (parallel.hpp:267-341): AccVec / DistVec are distinct RAII device-vector
// handles, status codes are rethrown as exception classes.
//
// BasicGpuBackend<Params, Errors> is parametrised on the parameter struct that
// params() returns and on the exception policy.  GpuBackend uses this
// header's own CycleParams and exception classes (standalone builds);
// include/patchmg_gpu_reference.hpp binds patchmg::CycleParams and the
// reference's patchmg:: exceptions (errors.hpp:9-56), so the reference's own
// templates -- patchmg::pcg_generic / mg_precondition / mg_cycle_generic from
// multigrid.hpp:120-189, compiled unchanged -- drive it
// (oracle/ref_templates/pcg_ref_templates.cpp, tests/test_gpu_cpp_dropin.py).
// The restated templates at the end of this header are for builds without the
// reference's headers.
#pragma once

#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pmg_cuda.h"

namespace patchmg_gpu {

struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct DefinitenessError : Error { using Error::Error; };
struct DecompositionError : Error { using Error::Error; };
struct DivergenceError : Error { using Error::Error; };
struct TransportError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

// status code -> exception (this header's classes)
inline void check(int rc, const char* msg) {
  switch (rc) {
    case PMG_OK: return;
    case PMG_ERR_CONFIG: throw ConfigError(msg);
    case PMG_ERR_DIVERGENCE: throw DivergenceError(msg);
    case PMG_ERR_TRANSPORT: throw TransportError(msg);
    case PMG_ERR_DOMAIN: throw DomainError(msg);
    case PMG_ERR_DEFINITENESS: throw DefinitenessError(msg);
    case PMG_ERR_DECOMPOSITION: throw DecompositionError(msg);
    case PMG_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

struct NativeErrors {
  static void raise(int rc, const char* msg) { check(rc, msg); }
};

struct CycleParams {  // multigrid.hpp:21-27
  int nu = 1, mu = 1;
  double tau = 0.25, sigma_scale = 0.2;
  bool damp_coarse = false;
};

template <int Form, class Errors = NativeErrors>
class DeviceVector {  // AccumulatedVector / DistributedVector, parallel.hpp:169-260
 public:
  DeviceVector() = default;
  DeviceVector(pmg_ctx* ctx, int level) : ctx_(ctx), level_(level) {
    pmg_vec* v = nullptr;
    Errors::raise(pmg_vec_create(ctx, level, &v), pmg_last_error(ctx));
    v_ = v;
  }
  DeviceVector(const DeviceVector& o) : DeviceVector(o.ctx_, o.level_) {
    Errors::raise(pmg_vec_copy(ctx_, o.v_, v_), pmg_last_error(ctx_));
  }
  DeviceVector& operator=(const DeviceVector& o) {
    if (this != &o) {
      if (!v_ || level_ != o.level_) {
        DeviceVector tmp(o.ctx_, o.level_);
        swap(tmp);
      }
      Errors::raise(pmg_vec_copy(ctx_, o.v_, v_), pmg_last_error(ctx_));
    }
    return *this;
  }
  DeviceVector(DeviceVector&& o) noexcept { swap(o); }
  DeviceVector& operator=(DeviceVector&& o) noexcept {
    swap(o);
    return *this;
  }
  ~DeviceVector() {
    if (v_) pmg_vec_free(v_);
  }
  void swap(DeviceVector& o) noexcept {
    std::swap(ctx_, o.ctx_);
    std::swap(v_, o.v_);
    std::swap(level_, o.level_);
  }
  pmg_vec* get() const { return v_; }
  int level() const { return level_; }
  static constexpr int form = Form;

 private:
  pmg_ctx* ctx_ = nullptr;
  pmg_vec* v_ = nullptr;
  int level_ = -1;
};

template <class Params = CycleParams, class Errors = NativeErrors>
class BasicGpuBackend {
 public:
  using AccVec = DeviceVector<PMG_ACCUMULATED, Errors>;
  using DistVec = DeviceVector<PMG_DISTRIBUTED, Errors>;

  BasicGpuBackend(const pmg_hierarchy_desc& h, int device = 0, const pmg_comm_desc* comm = nullptr) {
    prm_.nu = h.params.nu;
    prm_.mu = h.params.mu;
    prm_.tau = h.params.tau;
    prm_.sigma_scale = h.params.sigma_scale;
    prm_.damp_coarse = h.params.damp_coarse != 0;
    finest_ = h.num_levels - 1;
    Errors::raise(pmg_ctx_create(&h, device, comm, &ctx_), pmg_last_error(nullptr));
  }
  BasicGpuBackend(const BasicGpuBackend&) = delete;
  BasicGpuBackend& operator=(const BasicGpuBackend&) = delete;
  ~BasicGpuBackend() { pmg_ctx_destroy(ctx_); }

  const Params& params() const { return prm_; }
  int finest_level() const { return finest_; }
  pmg_ctx* ctx() const { return ctx_; }

  AccVec zero_acc(int level) const { return AccVec(ctx_, level); }
  DistVec apply_op(int level, const AccVec& u) const {
    DistVec out(ctx_, level);
    ok(pmg_apply_op(ctx_, level, u.get(), out.get()));
    return out;
  }
  DistVec residual(int level, const DistVec& f, const AccVec& u) const {
    DistVec out(ctx_, level);
    ok(pmg_residual(ctx_, level, f.get(), u.get(), out.get()));
    return out;
  }
  AccVec accumulate(int level, const DistVec& r) const {
    AccVec out(ctx_, level);
    ok(pmg_accumulate(ctx_, level, r.get(), out.get()));
    return out;
  }
  AccVec smooth(int level, const DistVec& r) const {
    AccVec out(ctx_, level);
    ok(pmg_smooth(ctx_, level, r.get(), out.get()));
    return out;
  }
  DistVec restrict_residual(int level, const DistVec& r) const {
    DistVec out(ctx_, level - 1);
    ok(pmg_restrict(ctx_, level, r.get(), out.get()));
    return out;
  }
  void add_prolonged(int level, const AccVec& coarse, double c, AccVec& u) const {
    ok(pmg_add_prolonged(ctx_, level, coarse.get(), c, u.get()));
  }
  AccVec coarse_solve(const DistVec& r) const {
    AccVec out(ctx_, 0);
    ok(pmg_coarse_solve(ctx_, r.get(), out.get()));
    return out;
  }
  double dot(int level, const DistVec& a, const AccVec& b) const {
    double d = 0.0;
    ok(pmg_dot(ctx_, level, a.get(), b.get(), &d));
    return d;
  }
  void axpy_acc(double a, const AccVec& x, AccVec& y) const { ok(pmg_axpy(ctx_, a, x.get(), y.get())); }
  void axpy_dist(double a, const DistVec& x, DistVec& y) const { ok(pmg_axpy(ctx_, a, x.get(), y.get())); }
  void xpay_acc(const AccVec& z, double beta, AccVec& p) const { ok(pmg_xpay(ctx_, z.get(), beta, p.get())); }

  // conversions (parallel.cpp:428-468)
  AccVec to_accumulated(int level, const std::vector<double>& g) const {
    AccVec v(ctx_, level);
    ok(pmg_vec_upload(ctx_, v.get(), PMG_ACCUMULATED, g.data(), int64_t(g.size())));
    return v;
  }
  DistVec to_distributed_owner(int level, const std::vector<double>& g) const {
    DistVec v(ctx_, level);
    ok(pmg_vec_upload(ctx_, v.get(), PMG_DISTRIBUTED, g.data(), int64_t(g.size())));
    return v;
  }
  template <int F>
  std::vector<double> gather_global(int level, const DeviceVector<F, Errors>& v, int64_t n) const {
    std::vector<double> out(static_cast<size_t>(n));
    ok(pmg_vec_download(ctx_, v.get(), F, out.data(), n));
    return out;
  }

 private:
  void ok(int rc) const { Errors::raise(rc, pmg_last_error(ctx_)); }
  pmg_ctx* ctx_ = nullptr;
  Params prm_;
  int finest_ = 0;
};

using GpuBackend = BasicGpuBackend<>;

// ---- the reference's templates, restated against the concept only, for
// builds without the reference's headers.  A nested namespace keeps them out
// of argument-dependent lookup, so a TU that also includes the reference's
// multigrid.hpp calls patchmg::pcg_generic & co. unambiguously.
namespace generic {

template <class B>
void mg_cycle_generic(const B& b, int level, typename B::AccVec& u, const typename B::DistVec& f) {
  const auto& prm = b.params();
  for (int i = 0; i < prm.nu; ++i) {
    typename B::AccVec z = b.smooth(level, b.residual(level, f, u));
    b.axpy_acc(prm.tau, z, u);
  }
  typename B::DistVec rc = b.restrict_residual(level, b.residual(level, f, u));
  typename B::AccVec p;
  if (level == 1) {
    p = b.coarse_solve(rc);
  } else {
    p = b.zero_acc(level - 1);
    for (int i = 0; i < prm.mu; ++i) mg_cycle_generic(b, level - 1, p, rc);
  }
  b.add_prolonged(level, p, prm.damp_coarse ? prm.tau : 1.0, u);
  for (int i = 0; i < prm.nu; ++i) {
    typename B::AccVec z = b.smooth(level, b.residual(level, f, u));
    b.axpy_acc(prm.tau, z, u);
  }
}

template <class B>
typename B::AccVec mg_precondition(const B& b, const typename B::DistVec& r) {
  typename B::AccVec z = b.zero_acc(b.finest_level());
  mg_cycle_generic(b, b.finest_level(), z, r);
  return z;
}

template <class B, class P>
typename B::AccVec pcg_generic(const B& b, const typename B::DistVec& f, double tol, int max_iter, const P& precond,
                               std::vector<double>& history) {
  const int L = b.finest_level();
  typename B::AccVec u = b.zero_acc(L);
  typename B::DistVec r = f;
  auto norm2 = [&](const typename B::DistVec& v) { return std::sqrt(b.dot(L, v, b.accumulate(L, v))); };
  const double r0 = norm2(r);
  history.clear();
  history.push_back(r0);
  if (r0 == 0.0) return u;
  typename B::AccVec z = precond(r);
  typename B::AccVec p = z;
  double rz = b.dot(L, r, z);
  for (int k = 1; k <= max_iter; ++k) {
    typename B::DistVec Ap = b.apply_op(L, p);
    const double pAp = b.dot(L, Ap, p);
    if (!(pAp > 0.0)) throw DefinitenessError("pcg: search direction with nonpositive energy");
    const double alpha = rz / pAp;
    b.axpy_acc(alpha, p, u);
    b.axpy_dist(-alpha, Ap, r);
    const double rn = norm2(r);
    history.push_back(rn);
    if (rn <= tol * r0) return u;
    z = precond(r);
    const double rz_next = b.dot(L, r, z);
    b.xpay_acc(z, rz_next / rz, p);
    rz = rz_next;
  }
  throw DivergenceError("pcg: no convergence within the iteration limit");
}

}  // namespace generic
}  // namespace patchmg_gpu
