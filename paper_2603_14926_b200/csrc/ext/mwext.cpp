// mwext.cpp — the PyTorch extension over the C-ABI (include/mwgpu.h).
//
// The Python package reaches the hot entry points of libmwgpu.so through
// this module: each function takes torch CUDA tensors, validates them
// (float64 planes, unit lane stride, one device, shapes), makes the
// operands' device current for the launch (CUDAGuard), takes torch's
// current stream on that device, and calls the C entry point -- one
// pybind call per operation instead of a ctypes call with 10-20 converted
// arguments.  Status codes become the reference's exceptions: MW_ERR_INVALID
// -> ValueError, MW_ERR_UNSUPPORTED -> NotImplementedError, CUDA errors ->
// RuntimeError.  No CPU fallback: a CPU tensor is an error.
//
// Plane convention (as the C-ABI): operand plane c starts at
// data_ptr + c * stride(0); lanes are contiguous (stride(-1) == 1), so
// column slices x[:, lo:hi] of a wider batch pass without a copy.
#include <torch/extension.h>

#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGraphsC10Utils.h>
#include <c10/cuda/CUDAGuard.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/mwgpu.h"

namespace py = pybind11;

namespace {

[[noreturn]] void raise_status(int rc, const char* what) {
  if (rc == MW_ERR_INVALID) throw py::value_error(std::string(what) + ": invalid arguments");
  if (rc == MW_ERR_UNSUPPORTED) {
    PyErr_SetString(PyExc_NotImplementedError,
                    (std::string(what) + ": no device kernel for this (k, variant) (no CPU fallback)").c_str());
    throw py::error_already_set();
  }
  const char* msg = mw_status_string(rc);
  throw std::runtime_error(std::string(what) + ": CUDA error " + std::to_string(rc) + ": " +
                           (msg ? msg : "?"));
}

inline void check(int rc, const char* what) {
  if (rc != MW_OK) raise_status(rc, what);
}

// K-word planes: CUDA float64, dim >= 2, plane dim 0, contiguous lanes.
void require_planes(const at::Tensor& t, const char* name, int64_t k, const c10::Device& dev) {
  if (!t.is_cuda())
    throw std::runtime_error(std::string("mwgpu: ") + name +
                             " must live on a CUDA device; the B200 path has no CPU fallback");
  if (t.scalar_type() != at::kDouble) throw py::value_error(std::string(name) + ": float64 planes required");
  if (t.device() != dev) throw py::value_error("mwgpu: operands on different devices");
  if (t.dim() < 2) throw py::value_error(std::string(name) + ": planes tensor (K, ...) expected");
  if (k >= 0 && t.size(0) != k) throw py::value_error("mixed word counts");
}

// The reference's argument errors come first, whatever the device
// (batch.py:197-201): mixed word counts, then mixed lane widths.
void check_pair(const at::Tensor& a, const at::Tensor& b) {
  if (a.dim() >= 1 && b.dim() >= 1 && a.size(0) != b.size(0)) throw py::value_error("mixed word counts");
  if (a.dim() == 2 && b.dim() == 2 && a.size(1) != b.size(1)) throw py::value_error("mixed lane widths");
}

// (K, W) planes with unit lane stride; returns the plane stride.
int64_t lane_planes(const at::Tensor& t, const char* name, int64_t k, const c10::Device& dev) {
  require_planes(t, name, k, dev);
  if (t.dim() != 2) throw py::value_error(std::string(name) + ": (K, lanes) planes expected");
  if (t.size(1) > 1 && t.stride(1) != 1) throw py::value_error(std::string(name) + ": lanes must be contiguous");
  if (t.size(0) > 1 && t.stride(0) < t.size(1)) throw py::value_error(std::string(name) + ": planes overlap");
  return t.size(0) > 1 ? t.stride(0) : t.size(1);
}

// Fully contiguous planes (matrices / coefficient arrays).
void contiguous_planes(const at::Tensor& t, const char* name, int64_t k, const c10::Device& dev) {
  require_planes(t, name, k, dev);
  if (!t.is_contiguous()) throw py::value_error(std::string(name) + ": planes tensor must be contiguous");
}

inline void* stream_of(const c10::Device& dev) {
  return reinterpret_cast<void*>(at::cuda::getCurrentCUDAStream(dev.index()).stream());
}

inline double* dptr(const at::Tensor& t) { return t.data_ptr<double>(); }

mw_tuning tuning_from(int64_t gemm_tile, int64_t dot_cluster, int64_t dk_tree_roots, int64_t dk_exact_roots,
                      int64_t dk_exact_split) {
  mw_tuning t;
  mw_tuning_defaults(&t);
  if (gemm_tile != INT64_MIN) t.gemm_tile = (int)gemm_tile;
  if (dot_cluster != INT64_MIN) t.dot_cluster = (int)dot_cluster;
  if (dk_tree_roots != INT64_MIN) t.dk_tree_roots = (int)dk_tree_roots;
  if (dk_exact_roots != INT64_MIN) t.dk_exact_roots = (int)dk_exact_roots;
  if (dk_exact_split != INT64_MIN) t.dk_exact_split = (int)dk_exact_split;
  return t;
}

// ------------------------------------------------------------------ lanes
// op: 0 add, 1 sub, 2 mul, 3 div (batch.py:204-231, linalg._ew_sub).
at::Tensor ew(int64_t op, int64_t variant, const at::Tensor& a, const at::Tensor& b,
              c10::optional<at::Tensor> out) {
  check_pair(a, b);
  const c10::Device dev = a.device();
  const int64_t k = a.dim() > 0 ? a.size(0) : 0;
  const int64_t sa = lane_planes(a, "a", k, dev);
  const int64_t sb = lane_planes(b, "b", k, dev);
  const int64_t w = a.size(1);
  if (b.size(1) != w) throw py::value_error("mixed lane widths");
  at::Tensor o = out.has_value() ? *out : at::empty({k, w}, a.options());
  const int64_t so = lane_planes(o, "out", k, dev);
  if (o.size(1) != w) throw py::value_error("out: lane width mismatch");
  if (w == 0) return o;
  c10::cuda::CUDAGuard guard(dev);
  void* st = stream_of(dev);
  int rc;
  switch (op) {
    case 0: rc = mw_ew_add((int)k, (int)variant, dptr(a), sa, dptr(b), sb, dptr(o), so, w, st); break;
    case 1: rc = mw_ew_sub((int)k, (int)variant, dptr(a), sa, dptr(b), sb, dptr(o), so, w, st); break;
    case 2: rc = mw_ew_mul((int)k, (int)variant, dptr(a), sa, dptr(b), sb, dptr(o), so, w, st); break;
    case 3: rc = mw_ew_div((int)k, (int)variant, dptr(a), sa, dptr(b), sb, dptr(o), so, w, st); break;
    default: throw py::value_error("unknown lane op");
  }
  check(rc, "mw_ew");
  return o;
}

// y <- alpha x + y (batch_mul then batch_add, batch.py:204-213).
void axpy_(int64_t variant, const std::vector<double>& alpha, const at::Tensor& x, const at::Tensor& y) {
  check_pair(x, y);
  const c10::Device dev = x.device();
  const int64_t k = x.dim() > 0 ? x.size(0) : 0;
  if ((int64_t)alpha.size() != k) throw py::value_error("mixed word counts");
  const int64_t sx = lane_planes(x, "x", k, dev);
  const int64_t sy = lane_planes(y, "y", k, dev);
  const int64_t n = x.size(1);
  if (y.size(1) != n) throw py::value_error("mixed lane widths");
  if (n == 0) return;
  c10::cuda::CUDAGuard guard(dev);
  check(mw_axpy((int)k, (int)variant, alpha.data(), dptr(x), sx, dptr(y), sy, n, stream_of(dev)), "mw_axpy");
}

// ------------------------------------------------------------------- dot
// Workspace of the tree dot (ws[0] = the single-launch ticket, then block
// partials).  Eager calls reuse one zeroed buffer per (device, stream) --
// calls on one stream are serialised and every call leaves the ticket at
// zero; a call being captured into a CUDA graph gets its OWN zeroed buffer
// (owned by the graph's private pool through the returned tensor), so
// graphs replayed on different streams never share a ticket.
std::mutex g_ws_mu;
std::map<std::pair<int, void*>, at::Tensor> g_ws;
constexpr size_t WS_CACHE_MAX = 64;

at::Tensor dot_workspace(int64_t need, const c10::Device& dev, void* st, bool capturing) {
  need = std::max<int64_t>(need, 1);
  auto opts = at::TensorOptions().dtype(at::kDouble).device(dev);
  if (capturing) return at::zeros({need}, opts);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto key = std::make_pair((int)dev.index(), st);
  auto it = g_ws.find(key);
  if (it != g_ws.end() && it->second.numel() >= need) return it->second;
  if (g_ws.size() >= WS_CACHE_MAX) g_ws.clear();  // bounded: short-lived streams do not pile up
  at::Tensor ws = at::zeros({need}, opts);
  g_ws[key] = ws;
  return ws;
}

at::Tensor dot(int64_t variant, const at::Tensor& x, const at::Tensor& y, int64_t order,
               c10::optional<at::Tensor> out, int64_t dot_cluster) {
  check_pair(x, y);
  const c10::Device dev = x.device();
  const int64_t k = x.dim() > 0 ? x.size(0) : 0;
  const int64_t sx = lane_planes(x, "x", k, dev);
  const int64_t sy = lane_planes(y, "y", k, dev);
  const int64_t n = x.size(1);
  if (y.size(1) != n) throw py::value_error("mixed lane widths");
  at::Tensor o = out.has_value() ? *out : at::empty({k}, x.options());
  if (!o.is_cuda() || o.scalar_type() != at::kDouble || o.device() != dev || o.numel() < k || !o.is_contiguous())
    throw py::value_error("out: K contiguous float64 values on the operands' device expected");
  c10::cuda::CUDAGuard guard(dev);
  void* st = stream_of(dev);
  const int64_t need = order == MW_ORDER_TREE ? mw_dot_workspace((int)k, n) : 0;
  at::Tensor ws;
  double* wsp = nullptr;
  if (need > 0) {
    // 2..16 blocks run as one cluster, which never touches the workspace
    // (it is passed for the ticket-form fallback only)
    const int64_t nb = (n + 4095) / 4096;
    const bool cluster_path = dot_cluster != 0 && nb > 1 && nb <= 16;
    const bool capturing = c10::cuda::currentStreamCaptureStatusMayInitCtx() != c10::cuda::CaptureStatus::None;
    ws = dot_workspace(need, dev, st, capturing && !cluster_path);
    wsp = dptr(ws);
  }
  const mw_tuning t = tuning_from(INT64_MIN, dot_cluster, INT64_MIN, INT64_MIN, INT64_MIN);
  check(mw_dot_ex((int)k, (int)variant, dptr(x), sx, dptr(y), sy, n, wsp, dptr(o), (int)order, &t, st),
        "mw_dot");
  return o;
}

// ------------------------------------------------------------------ GEMV
// y = A[row0:row1] x (A: (K, m, n) contiguous planes).
at::Tensor gemv(int64_t variant, const at::Tensor& A, const at::Tensor& x, int64_t row0, int64_t row1,
                int64_t order, c10::optional<at::Tensor> out) {
  const c10::Device dev = A.device();
  const int64_t k = A.dim() > 0 ? A.size(0) : 0;
  contiguous_planes(A, "A", k, dev);
  if (A.dim() != 3) throw py::value_error("A: (K, rows, cols) planes expected");
  const int64_t m = A.size(1), n = A.size(2);
  const int64_t sx = lane_planes(x, "x", k, dev);
  if (x.size(1) != n) throw py::value_error("shape mismatch: A cols != x width");
  if (row1 < 0) row1 = m;
  if (row0 < 0 || row0 > row1 || row1 > m) throw py::value_error("row range outside the matrix");
  const int64_t rows = row1 - row0;
  at::Tensor o = out.has_value() ? *out : at::empty({k, rows}, A.options());
  const int64_t so = lane_planes(o, "out", k, dev);
  if (o.size(1) != rows) throw py::value_error("out: width != rows");
  if (rows == 0) return o;
  c10::cuda::CUDAGuard guard(dev);
  check(mw_gemv((int)k, (int)variant, dptr(A) + row0 * n, n, m * n, dptr(x), sx, dptr(o), so, rows, n, (int)order,
                stream_of(dev)),
        "mw_gemv");
  return o;
}

// ------------------------------------------------------------------ GEMM
// C[row0:row1] = A[row0:row1] B on (K, m, kd), (K, kd, n), (K, m, n).
void gemm(int64_t variant, const at::Tensor& A, const at::Tensor& B, const at::Tensor& C, int64_t row0,
          int64_t row1, int64_t gemm_tile) {
  const c10::Device dev = A.device();
  const int64_t k = A.dim() > 0 ? A.size(0) : 0;
  contiguous_planes(A, "A", k, dev);
  contiguous_planes(B, "B", k, dev);
  contiguous_planes(C, "C", k, dev);
  if (A.dim() != 3 || B.dim() != 3 || C.dim() != 3) throw py::value_error("gemm: (K, rows, cols) planes expected");
  const int64_t m = A.size(1), kd = A.size(2), n = B.size(2);
  if (B.size(1) != kd || C.size(1) != m || C.size(2) != n) throw py::value_error("gemm: shape mismatch");
  if (row1 < 0) row1 = m;
  if (row0 < 0 || row0 > row1 || row1 > m) throw py::value_error("row range outside the matrix");
  const int64_t rows = row1 - row0;
  if (rows == 0 || n == 0) return;
  c10::cuda::CUDAGuard guard(dev);
  const mw_tuning t = tuning_from(gemm_tile, INT64_MIN, INT64_MIN, INT64_MIN, INT64_MIN);
  check(mw_gemm_ex((int)k, (int)variant, dptr(A) + row0 * kd, kd, m * kd, dptr(B), n, kd * n, dptr(C) + row0 * n, n,
                   m * n, rows, n, kd, &t, stream_of(dev)),
        "mw_gemm");
}

// ---------------------------------------------------------------- Horner
// y[:, p0:p1] = Horner(coeffs, x[:, p0:p1]) (poly.py:89-96).
void horner(int64_t variant, const at::Tensor& coeffs, const at::Tensor& x, const at::Tensor& y, int64_t p0,
            int64_t p1) {
  const c10::Device dev = x.device();
  const int64_t k = x.dim() > 0 ? x.size(0) : 0;
  contiguous_planes(coeffs, "coeffs", k, dev);
  if (coeffs.dim() != 2 || coeffs.size(1) < 1) throw py::value_error("coeffs: (K, degree+1) planes expected");
  const int64_t sx = lane_planes(x, "x", k, dev);
  const int64_t sy = lane_planes(y, "y", k, dev);
  const int64_t npts = x.size(1);
  if (y.size(1) != npts) throw py::value_error("mixed lane widths");
  if (p1 < 0) p1 = npts;
  if (p0 < 0 || p0 > p1 || p1 > npts) throw py::value_error("point range outside the batch");
  if (p1 == p0) return;
  c10::cuda::CUDAGuard guard(dev);
  check(mw_horner((int)k, (int)variant, dptr(coeffs), coeffs.size(1), coeffs.size(1) - 1, dptr(x) + p0, sx,
                  dptr(y) + p0, sy, p1 - p0, stream_of(dev)),
        "mw_horner");
}

// ------------------------------------------------------------ DK sweep
// Roots [i0, i1) of the frozen state (zre, zim: (K, n)) -> out planes at the
// same indices; step_mag (n), flag (int32, INT32_MAX beforehand).  The tree
// order takes a stream-ordered workspace from the caching allocator.
void dk_sweep(int64_t variant, const at::Tensor& coeffs, const at::Tensor& zre, const at::Tensor& zim,
              const at::Tensor& out_re, const at::Tensor& out_im, const at::Tensor& step_mag,
              const at::Tensor& flag, bool exact_order, int64_t i0, int64_t i1, int64_t dk_tree_roots,
              int64_t dk_exact_roots, int64_t dk_exact_split, c10::optional<at::Tensor> max_bits) {
  const c10::Device dev = zre.device();
  const int64_t k = zre.dim() > 0 ? zre.size(0) : 0;
  for (auto* p : {&coeffs, &zre, &zim, &out_re, &out_im}) contiguous_planes(*p, "dk planes", k, dev);
  const int64_t n = zre.size(1);
  if (coeffs.size(1) != n || zim.size(1) != n || out_re.size(1) != n || out_im.size(1) != n)
    throw py::value_error("state size does not match the polynomial degree");
  if (!step_mag.is_cuda() || step_mag.scalar_type() != at::kDouble || step_mag.numel() < n ||
      !step_mag.is_contiguous() || step_mag.device() != dev)
    throw py::value_error("step_mag: n contiguous float64 on the state's device expected");
  if (!flag.is_cuda() || flag.scalar_type() != at::kInt || flag.numel() < 1 || flag.device() != dev)
    throw py::value_error("flag: int32 device scalar expected");
  if (i1 < 0) i1 = n;
  unsigned long long* maxp = nullptr;
  if (max_bits.has_value()) {
    const at::Tensor& mb = *max_bits;
    if (!mb.is_cuda() || mb.scalar_type() != at::kLong || mb.numel() < 2 || !mb.is_contiguous() ||
        mb.device() != dev)
      throw py::value_error("max_bits: two contiguous int64 on the state's device expected");
    maxp = reinterpret_cast<unsigned long long*>(mb.data_ptr<int64_t>());
  }
  c10::cuda::CUDAGuard guard(dev);
  void* st = stream_of(dev);
  at::Tensor ws;
  double* wsp = nullptr;
  if (!exact_order && i1 > i0) {
    ws = at::empty({std::max<int64_t>(mw_dk_sweep_workspace((int)k, i0, i1), 1)}, zre.options());
    wsp = dptr(ws);
  }
  const mw_tuning t = tuning_from(INT64_MIN, INT64_MIN, dk_tree_roots, dk_exact_roots, dk_exact_split);
  check(mw_dk_sweep_ex((int)k, (int)variant, dptr(coeffs), n, n, dptr(zre), dptr(zim), n, i0, i1, dptr(out_re),
                       dptr(out_im), n, dptr(step_mag), flag.data_ptr<int>(), exact_order ? 1 : 0, wsp, maxp, &t,
                       st),
        "mw_dk_sweep");
}

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.doc() = "PyTorch extension over libmwgpu.so (include/mwgpu.h): hot entry points on torch tensors";
  const int64_t D = INT64_MIN;  // "library default" for a tuning field
  m.def("ew", &ew, py::arg("op"), py::arg("variant"), py::arg("a"), py::arg("b"), py::arg("out") = py::none());
  m.def("axpy_", &axpy_, py::arg("variant"), py::arg("alpha"), py::arg("x"), py::arg("y"));
  m.def("dot", &dot, py::arg("variant"), py::arg("x"), py::arg("y"), py::arg("order"), py::arg("out") = py::none(),
        py::arg("dot_cluster") = D);
  m.def("gemv", &gemv, py::arg("variant"), py::arg("A"), py::arg("x"), py::arg("row0") = 0, py::arg("row1") = -1,
        py::arg("order") = MW_ORDER_TREE, py::arg("out") = py::none());
  m.def("gemm", &gemm, py::arg("variant"), py::arg("A"), py::arg("B"), py::arg("C"), py::arg("row0") = 0,
        py::arg("row1") = -1, py::arg("gemm_tile") = D);
  m.def("horner", &horner, py::arg("variant"), py::arg("coeffs"), py::arg("x"), py::arg("y"), py::arg("p0") = 0,
        py::arg("p1") = -1);
  m.def("dk_sweep", &dk_sweep, py::arg("variant"), py::arg("coeffs"), py::arg("zre"), py::arg("zim"),
        py::arg("out_re"), py::arg("out_im"), py::arg("step_mag"), py::arg("flag"), py::arg("exact_order"),
        py::arg("i0") = 0, py::arg("i1") = -1, py::arg("dk_tree_roots") = D, py::arg("dk_exact_roots") = D,
        py::arg("dk_exact_split") = D, py::arg("max_bits") = py::none());
  m.def("version", []() { return std::string(mw_version()); });
}
