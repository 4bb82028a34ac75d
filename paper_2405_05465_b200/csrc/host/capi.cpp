// capi.cpp -- the extern "C" boundary (include/ssg.h) over the C++ drop-in API.
//
// Exceptions never cross the ABI: servesim::Error -> 1 (message verbatim),
// InternalError -> 2, CUDA failures -> 3.
#include "ssg.h"

#include <cstdlib>
#include <cstring>
#include <functional>

#include "runtime.h"
#include "servesim_b200.hpp"

using namespace servesim;

struct ssg_estimator {
  EstimatorModel model;
};

namespace ssg {
void launch_predict(const DeviceEstimator& de, int64_t n, const int32_t* slots, int32_t uniform,
                    const double* f0, const double* f1, double* out,
                    unsigned long long* first_error, cudaStream_t s);
[[noreturn]] void raise_predict_error(const EstimatorModel& est, unsigned long long word,
                                      const int32_t* slots_host, int32_t uniform,
                                      const double* f0_host, const double* f1_host);
}  // namespace ssg

namespace {

void set_status(ssg_status* st, int code, const char* msg) {
  if (!st) return;
  st->code = code;
  std::strncpy(st->message, msg ? msg : "", sizeof(st->message) - 1);
  st->message[sizeof(st->message) - 1] = '\0';
}

int guarded(ssg_status* st, const std::function<void()>& body) {
  try {
    body();
    set_status(st, SSG_STATUS_OK, "");
    return SSG_STATUS_OK;
  } catch (const Error& e) {
    set_status(st, SSG_STATUS_INPUT, e.what());
    return SSG_STATUS_INPUT;
  } catch (const ssg::CudaError& e) {
    set_status(st, SSG_STATUS_CUDA, e.what());
    return SSG_STATUS_CUDA;
  } catch (const InternalError& e) {
    set_status(st, SSG_STATUS_INTERNAL, e.what());
    return SSG_STATUS_INTERNAL;
  } catch (const std::exception& e) {
    set_status(st, SSG_STATUS_INTERNAL, e.what());
    return SSG_STATUS_INTERNAL;
  }
}

char* dup_text(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw InternalError("out of host memory");
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  if (len) *len = s.size();
  return p;
}

// Grow-only staging buffers for the host-buffer entry points.
struct Staging {
  ssg::DeviceBuffer<int32_t> slots;
  ssg::DeviceBuffer<double> f0, f1, out;
  ssg::DeviceBuffer<unsigned long long> err;
};
Staging& staging() {
  static Staging s;
  return s;
}

void predict_host(const EstimatorModel& est, size_t n, const int32_t* slots, int32_t uniform,
                  const double* f0, const double* f1, double* out) {
  if (n == 0) return;
  const auto& de = est.device();
  auto& ctx = ssg::context();
  auto& S = staging();
  cudaStream_t s = ctx.stream;
  if (slots) S.slots.upload(slots, n, s);
  S.f0.upload(f0, n, s);
  if (f1) S.f1.upload(f1, n, s);
  S.out.resize(n);
  unsigned long long none = SSG_NO_ERROR, word = 0;
  S.err.upload(&none, 1, s);
  ssg::launch_predict(de, static_cast<int64_t>(n), slots ? S.slots.ptr : nullptr, uniform, S.f0.ptr,
                      f1 ? S.f1.ptr : nullptr, S.out.ptr, S.err.ptr, s);
  S.out.download(out, n, s);
  S.err.download(&word, 1, s);
  ssg::cuda_check(cudaStreamSynchronize(s), "predict");
  if (word != SSG_NO_ERROR) ssg::raise_predict_error(est, word, slots, uniform, f0, f1);
}

}  // namespace

extern "C" {

int ssg_init(int device, ssg_status* st) {
  return guarded(st, [&] { ssg::init_context(device); });
}

int ssg_shutdown(void) {
  ssg::shutdown_context();
  return SSG_STATUS_OK;
}

int ssg_math_variant(void) {
  try {
    return ssg::probe_host_math_variant();
  } catch (...) {
    return -1;
  }
}

const char* ssg_version(void) { return "ssg 0.1 sm_100a"; }

void ssg_free(void* p) { std::free(p); }

int ssg_estimator_from_json(const char* json, size_t len, ssg_estimator** out, ssg_status* st) {
  return guarded(st, [&] {
    auto* e = new ssg_estimator{EstimatorModel::from_json(std::string(json, len))};
    *out = e;
  });
}

int ssg_estimator_train(const char* model_spec_json, const char* device_json, const int64_t* tps,
                        size_t n_tps, const char* regressor, uint64_t seed, ssg_estimator** out,
                        ssg_status* st) {
  return guarded(st, [&] {
    ModelSpec spec = parse_model_spec(model_spec_json);
    DeviceProfile dev = parse_device_profile(device_json);
    std::vector<std::int64_t> tp(tps, tps + n_tps);
    TrainConfig cfg;
    cfg.seed = seed;
    cfg.regressor = regressor ? regressor : "interp";
    auto* e = new ssg_estimator{train(generate_synthetic_profile(spec, dev, tp), cfg)};
    *out = e;
  });
}

int ssg_estimator_to_json(const ssg_estimator* e, char** out, size_t* len, ssg_status* st) {
  return guarded(st, [&] { *out = dup_text(e->model.to_json(), len); });
}

void ssg_estimator_free(ssg_estimator* e) { delete e; }

int32_t ssg_estimator_slot(const ssg_estimator* e, int32_t op, int64_t tp) {
  try {
    return e->model.device().slot(static_cast<OpName>(op), tp);
  } catch (...) {
    return -1;
  }
}

int64_t ssg_estimator_device_bytes(const ssg_estimator* e, ssg_status* st) {
  int64_t b = -1;
  guarded(st, [&] { b = static_cast<int64_t>(e->model.device().bytes); });
  return b;
}

int ssg_predict(const ssg_estimator* e, int32_t op, int64_t tp, size_t n, const double* f0,
                const double* f1, double* out, ssg_status* st) {
  return guarded(st, [&] {
    const auto& m = e->model.find(static_cast<OpName>(op), tp);
    require(m.schema.size() == 1 || f1 != nullptr,
            "estimator: query for " + to_string(OpModelKey{static_cast<OpName>(op), tp}) +
                " missing feature " + m.schema.back());
    const int32_t slot = e->model.device().slot(static_cast<OpName>(op), tp);
    predict_host(e->model, n, nullptr, slot, f0, m.schema.size() > 1 ? f1 : nullptr, out);
  });
}

int ssg_predict_mixed(const ssg_estimator* e, size_t n, const int32_t* slots, const double* f0,
                      const double* f1, double* out, ssg_status* st) {
  return guarded(st, [&] {
    const auto& de = e->model.device();
    for (size_t i = 0; i < n; ++i)
      require(slots[i] >= 0 && slots[i] < de.view.nmodels,
              "predict: query " + std::to_string(i) + " has no trained model slot");
    predict_host(e->model, n, slots, 0, f0, f1, out);
  });
}

int ssg_predict_device(const ssg_estimator* e, size_t n, const int32_t* d_slots,
                       int32_t uniform_slot, const double* d_f0, const double* d_f1, double* d_out,
                       unsigned long long* d_first_error, void* stream, ssg_status* st) {
  return guarded(st, [&] {
    const auto& de = e->model.device();
    require(d_slots || (uniform_slot >= 0 && uniform_slot < de.view.nmodels),
            "predict: invalid model slot");
    ssg::launch_predict(de, static_cast<int64_t>(n), d_slots, uniform_slot, d_f0, d_f1, d_out,
                        d_first_error, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
