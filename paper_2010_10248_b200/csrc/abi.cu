// extern "C" entry points of libstb200.so (declared in include/stb200.h).
// Every entry converts C++ exceptions / CUDA errors into a status code and a
// thread-local message; nothing throws across the ABI.
#include <cstdio>
#include <cstring>
#include <vector>
#include <memory>
#include <new>
#include <string>

#include "stb_internal.cuh"

namespace stb {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace stb

#define STB_API extern "C" __attribute__((visibility("default")))

#define STB_GUARD(...)                                         \
  try {                                                        \
    __VA_ARGS__;                                                    \
    return STB_OK;                                             \
  } catch (const stb::Error& e) {                              \
    stb::set_error(e.what());                                  \
    return e.code;                                             \
  } catch (const std::bad_alloc&) {                            \
    stb::set_error("host allocation failed");                  \
    return STB_ERR_NOMEM;                                      \
  } catch (const std::exception& e) {                          \
    stb::set_error(e.what());                                  \
    return STB_ERR_CUDA;                                       \
  } catch (...) {                                              \
    stb::set_error("unknown error");                           \
    return STB_ERR_CUDA;                                       \
  }

namespace {

void check_geometry(const stb_geometry* g) {
  STB_REQUIRE(g != nullptr, STB_ERR_ARG, "geometry is NULL");
  for (int a = 0; a < 3; ++a) {
    STB_REQUIRE(g->shape[a] >= 1, STB_ERR_ARG, "every shape extent must be >= 1");
    STB_REQUIRE(g->spacing[a] > 0.0, STB_ERR_ARG, "every spacing must be > 0");
  }
}

void check_order(int so) {
  STB_REQUIRE(so % 2 == 0 && so >= 2 && so <= 16, STB_ERR_CONFIG,
              "space_order: must be even in [2, 16]");
}

void check_precision(int p) {
  STB_REQUIRE(p == 32 || p == 64, STB_ERR_CONFIG, "precision: must be 32 or 64");
}

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw stb::Error(STB_ERR_CUDA, std::string("no CUDA device available: ") +
                                       (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)));
}

}  // namespace

STB_API int stb_abi_version(void) { return STB_ABI_VERSION; }

STB_API const char* stb_last_error(void) { return stb::g_last_error.c_str(); }

STB_API int stb_device_count(int* count) {
  STB_GUARD({
    STB_REQUIRE(count != nullptr, STB_ERR_ARG, "count is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    *count = (e == cudaSuccess) ? n : 0;
    if (e != cudaSuccess) cudaGetLastError();
  })
}

STB_API int stb_set_device(int device) {
  STB_GUARD({ STB_CUDA(cudaSetDevice(device)); })
}

STB_API int stb_host_alloc(int64_t bytes, void** out) {
  STB_GUARD({
    STB_REQUIRE(out != nullptr && bytes > 0, STB_ERR_ARG, "stb_host_alloc: bad arguments");
    require_device();
    *out = stb::host_pinned_alloc((size_t)bytes);
    STB_REQUIRE(*out != nullptr, STB_ERR_NOMEM, "page-locked host allocation failed");
  })
}

STB_API int stb_host_free(void* p) {
  STB_GUARD({
    STB_REQUIRE(p == nullptr || stb::host_pinned_free(p), STB_ERR_ARG,
                "stb_host_free: not a block of stb_host_alloc");
  })
}

STB_API int stb_interp_stencils(const double* coords, int64_t n, const stb_geometry* g,
                                int64_t margin, int64_t* idx_out, double* w_out) {
  STB_GUARD({
    check_geometry(g);
    STB_REQUIRE(n >= 0, STB_ERR_ARG, "n must be >= 0");
    if (n == 0) return STB_OK;
    require_device();
    stb::DevBuf<double> c(n * 3), w(n * 8);
    stb::DevBuf<int64_t> idx(n * 24);
    c.upload(coords, n * 3);
    stb::stencils_compute(c.p, n, *g, margin, idx.p, w.p, 0);
    if (idx_out) idx.download(idx_out, n * 24);
    if (w_out) w.download(w_out, n * 8);
    STB_CUDA(cudaDeviceSynchronize());
  })
}

STB_API int stb_support_create(const double* coords, int64_t n, const stb_geometry* g,
                               int32_t keep_zero_weights, stb_support_t* out) {
  STB_GUARD({
    check_geometry(g);
    STB_REQUIRE(out != nullptr, STB_ERR_ARG, "out is NULL");
    STB_REQUIRE(n >= 0, STB_ERR_ARG, "n must be >= 0");
    require_device();
    auto h = std::make_unique<stb_support_s>();
    stb::support_build(h->s, coords, n, *g, keep_zero_weights != 0, 0);
    *out = h.release();
  })
}

STB_API int stb_support_from_points(const int64_t* points, int64_t n, const stb_geometry* g,
                                    stb_support_t* out) {
  STB_GUARD({
    check_geometry(g);
    STB_REQUIRE(out != nullptr, STB_ERR_ARG, "out is NULL");
    STB_REQUIRE(n >= 0, STB_ERR_ARG, "n must be >= 0");
    require_device();
    auto h = std::make_unique<stb_support_s>();
    stb::support_from_points(h->s, points, n, *g, 0);
    *out = h.release();
  })
}

STB_API int stb_support_info(stb_support_t s, int64_t* n_affected, int64_t* n_entries) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    if (n_affected) *n_affected = s->s.K;
    if (n_entries) *n_entries = s->s.M;
  })
}

STB_API int stb_support_points(stb_support_t s, int64_t* points) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    stb::support_points_host(s->s, points, 0);
  })
}

STB_API int stb_support_compress(stb_support_t s, int32_t* nnz_mask, int64_t* row_ptr,
                                 int64_t* flat_z, int32_t* flat_id) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    stb::support_compress_host(s->s, nnz_mask, row_ptr, flat_z, flat_id, 0);
  })
}

STB_API int stb_support_masks(stb_support_t s, uint8_t* sm, int32_t* sid) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    stb::support_masks_host(s->s, sm, sid, 0);
  })
}

STB_API int stb_support_entries(stb_support_t s, int64_t* entry_points, int64_t* entry_owner,
                                double* entry_w) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    stb::support_entries_host(s->s, entry_points, entry_owner, entry_w, 0);
  })
}

STB_API int stb_support_decompose(stb_support_t s, const double* wavelets, int64_t nt_w,
                                  const double* scale, int64_t nt, double* src_dcmp) {
  STB_GUARD({
    STB_REQUIRE(s != nullptr, STB_ERR_ARG, "support handle is NULL");
    STB_REQUIRE(nt >= nt_w, STB_ERR_ARG, "nt is shorter than the wavelet length");
    const auto& sp = s->s;
    if (sp.K == 0 || nt == 0) return STB_OK;
    stb::DevBuf<double> wav(nt_w * sp.n_points), sc(sp.n_points), out(nt * sp.K);
    wav.upload(wavelets, nt_w * sp.n_points);
    sc.upload(scale, sp.n_points);
    stb::support_decompose_dev(sp, wav.p, nt_w, sc.p, nt, out.p, 0);
    out.download(src_dcmp, nt * sp.K);
    STB_CUDA(cudaDeviceSynchronize());
  })
}

STB_API int stb_support_destroy(stb_support_t s) {
  STB_GUARD({ delete s; })
}

STB_API int stb_acoustic_create(const stb_acoustic_desc* d, stb_prop_t* out) {
  STB_GUARD({
    STB_REQUIRE(d != nullptr && out != nullptr, STB_ERR_ARG, "NULL argument");
    check_geometry(&d->geom);
    check_order(d->space_order);
    check_precision(d->precision);
    require_device();
    *out = make_acoustic(*d);
  })
}

STB_API int stb_elastic_create(const stb_elastic_desc* d, stb_prop_t* out) {
  STB_GUARD({
    STB_REQUIRE(d != nullptr && out != nullptr, STB_ERR_ARG, "NULL argument");
    check_geometry(&d->geom);
    check_order(d->space_order);
    check_precision(d->precision);
    require_device();
    *out = make_elastic(*d);
  })
}

STB_API int stb_tti_create(const stb_tti_desc* d, stb_prop_t* out) {
  STB_GUARD({
    STB_REQUIRE(d != nullptr && out != nullptr, STB_ERR_ARG, "NULL argument");
    check_geometry(&d->geom);
    check_order(d->space_order);
    check_precision(d->precision);
    require_device();
    *out = make_tti(*d);
  })
}

STB_API int stb_prop_set_receiver_field(stb_prop_t p, int32_t field) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->set_receiver_field(field);
  })
}

STB_API int stb_prop_set_damping(stb_prop_t p, const double* fx, const double* fy,
                                 const double* fz) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    const double* t[3] = {fx, fy, fz};
    p->set_damping(t);
  })
}

STB_API int stb_prop_stream(stb_prop_t p, void** stream) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && stream != nullptr, STB_ERR_ARG, "NULL argument");
    *stream = p->stream();
  })
}

STB_API int stb_prop_async_begin(stb_prop_t p, int64_t t0, int64_t nsteps) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->async_begin(t0, nsteps);
  })
}

STB_API int stb_prop_step_async(stb_prop_t p, int64_t t, int32_t kb, int64_t x_lo, int64_t x_hi) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->step_async(t, kb, x_lo, x_hi);
  })
}

STB_API int stb_prop_half_step_async(stb_prop_t p, int64_t t, int32_t phase, int64_t x_lo,
                                     int64_t x_hi) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->half_step_async(t, phase, x_lo, x_hi);
  })
}

STB_API int stb_prop_step_async_peers(stb_prop_t p, int64_t t, int64_t x_lo, int64_t x_hi,
                                      const stb_peer_halo* peers) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && peers != nullptr, STB_ERR_ARG, "NULL argument");
    p->step_async_peers(t, x_lo, x_hi, peers);
  })
}

STB_API int stb_prop_gather_async(stb_prop_t p, int64_t t, int32_t kb) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->gather_async(t, kb);
  })
}

STB_API int stb_prop_async_finish(stb_prop_t p, double* rec_out, int64_t* bad_step) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->async_finish(rec_out, bad_step);
  })
}

STB_API int stb_prop_write_snapshot(stb_prop_t p, int32_t field, int64_t t, const char* path) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && path != nullptr, STB_ERR_ARG, "NULL argument");
    STB_REQUIRE(t >= 0 && t <= (int64_t)UINT32_MAX, STB_ERR_ARG, "time index out of range");
    int64_t shape[3];
    int elem = 0;
    p->field_info(shape, &elem);
    STB_REQUIRE(shape[0] <= INT32_MAX && shape[1] <= INT32_MAX && shape[2] <= INT32_MAX,
                STB_ERR_ARG, "field too large for the snapshot header");
    std::vector<unsigned char> buf((size_t)(shape[0] * shape[1] * shape[2]) * elem);
    p->read_field(field, t, buf.data());
    unsigned char head[32] = {0};
    std::memcpy(head, "STBSNAP\0", 8);
    const uint32_t bits = (uint32_t)(8 * elem), tt = (uint32_t)t;
    const int32_t dims[3] = {(int32_t)shape[0], (int32_t)shape[1], (int32_t)shape[2]};
    std::memcpy(head + 8, &bits, 4);
    std::memcpy(head + 12, dims, 12);
    std::memcpy(head + 24, &tt, 4);
    std::FILE* f = std::fopen(path, "wb");
    STB_REQUIRE(f != nullptr, STB_ERR_ARG, std::string("cannot open ") + path);
    const bool ok = std::fwrite(head, 1, 32, f) == 32 &&
                    std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
    std::fclose(f);
    STB_REQUIRE(ok, STB_ERR_ARG, std::string("short write to ") + path);
  })
}

STB_API int stb_prop_set_sources(stb_prop_t p, stb_support_t s, const double* wavelets,
                                 int64_t nt_w, const double* scale, int64_t nt) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && s != nullptr, STB_ERR_ARG, "NULL handle");
    STB_REQUIRE(nt >= nt_w, STB_ERR_ARG, "nt is shorter than the wavelet length");
    p->set_sources(s->s, wavelets, nt_w, scale, nt);
  })
}

STB_API int stb_prop_set_receivers(stb_prop_t p, const double* coords, int64_t nrec) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    STB_REQUIRE(nrec >= 0, STB_ERR_ARG, "nrec must be >= 0");
    p->set_receivers(coords, nrec);
  })
}

STB_API int stb_prop_run(stb_prop_t p, int64_t t0, int64_t nsteps, int32_t time_height,
                         double* rec_out, int64_t* bad_step) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    STB_REQUIRE(t0 >= 0 && nsteps >= 0, STB_ERR_ARG, "t0 and nsteps must be >= 0");
    STB_REQUIRE(time_height >= 0, STB_ERR_PLAN, "time_height must be >= 1");
    p->run(t0, nsteps, time_height, rec_out, bad_step);
  })
}

STB_API int stb_prop_read_field(stb_prop_t p, int32_t field, int64_t t, void* out) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && out != nullptr, STB_ERR_ARG, "NULL argument");
    p->read_field(field, t, out);
  })
}

STB_API int stb_prop_level_ptr(stb_prop_t p, int32_t field, int64_t t, void** dev,
                               int64_t* plane_elems, int64_t* pitch_elems) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && dev != nullptr, STB_ERR_ARG, "NULL argument");
    p->level_ptr(field, t, dev, plane_elems, pitch_elems);
  })
}

STB_API int stb_prop_reset(stb_prop_t p) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->reset();
  })
}

STB_API int stb_prop_stats(stb_prop_t p, int64_t* launches, double* kernel_ms,
                           int64_t* updates, int64_t* all_launches, double* run_ms) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr, STB_ERR_ARG, "NULL handle");
    p->stats(launches, kernel_ms, updates, all_launches, run_ms);
  })
}

STB_API int stb_prop_describe(stb_prop_t p, int32_t time_height, char* buf, int64_t buflen) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && buf != nullptr && buflen > 0, STB_ERR_ARG, "NULL argument");
    const std::string s = p->describe(time_height);
    std::strncpy(buf, s.c_str(), (size_t)buflen - 1);
    buf[buflen - 1] = '\0';
  })
}

STB_API int stb_prop_max_time_height(stb_prop_t p, int32_t* k) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && k != nullptr, STB_ERR_ARG, "NULL argument");
    *k = p->max_time_height();
  })
}

STB_API int stb_prop_velocity_max(stb_prop_t p, double* vmax) {
  STB_GUARD({
    STB_REQUIRE(p != nullptr && vmax != nullptr, STB_ERR_ARG, "NULL argument");
    *vmax = p->velocity_max();
  })
}

STB_API int stb_prop_destroy(stb_prop_t p) {
  STB_GUARD({ delete p; })
}
