// Per-call latency of the reference-style single-query APIs on the GPU
// (EstimatorModel::predict, Regressor::predict).  Diagnostic; built by hand:
//   g++ -O2 -std=gnu++20 -Iinclude -I<json dir> tools/time_single_query.cpp \
//       -Lpaper_2405_05465_b200 -lssg -Wl,-rpath,$PWD/paper_2405_05465_b200 -o build/time_single_query
#include <chrono>
#include <cstdio>

#include "servesim_b200.hpp"
using namespace servesim;
int main() {
  ModelSpec spec = parse_model_spec(R"({"schema_version":1,"name":"llama2-7b","num_layers":32,"hidden_dim":4096,"num_q_heads":32,"num_kv_heads":32,"head_dim":128,"mlp_dim":11008,"vocab_size":32000,"max_context":4096,"param_bytes_per_element":2,"attention_variant":"mha"})");
  DeviceProfile dev = parse_device_profile(R"({"schema_version":1,"sku_name":"A100-80G","peak_flops":312e12,"mem_bandwidth":2.039e12,"link_bandwidth":3.0e11,"kernel_overhead":2e-6,"device_mem":80e9})");
  TrainConfig tc;
  auto est = train(generate_synthetic_profile(spec, dev, {1}), tc);
  double s = 0;
  for (int i = 0; i < 100; ++i) s += est.predict(OpName::MlpUpProj, 1, {{"num_tokens", 100.0 + i}});
  const int n = 20000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) s += est.predict(OpName::AttnDecode, 1, {{"num_tokens", 1.0 + i % 64}, {"kv_read_bytes", 524288.0 * (1 + i % 100)}});
  auto t1 = std::chrono::steady_clock::now();
  auto reg = regressor_from_json(est.to_json()["ops"]["attn_decode@tp1"]["regressor"]);
  std::vector<double> x{2.0, 13.0};
  for (int i = 0; i < 100; ++i) s += reg->predict(x);
  auto t2 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) { x[0] = 1.0 + (i % 50) * 0.1; s += reg->predict(x); }
  auto t3 = std::chrono::steady_clock::now();
  std::printf("EstimatorModel::predict %.2f us/call; Regressor::predict %.2f us/call (checksum %g)\n",
              std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
              std::chrono::duration<double, std::micro>(t3 - t2).count() / n, s);
}
