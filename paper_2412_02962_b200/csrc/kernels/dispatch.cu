// Kernel selection: tcgen05 (sm_100a tensor cores) for the bf16 contractions the TC kernels
// support, SIMT otherwise (fp32 parity mode, conv_in, odd shapes).
#include <atomic>
#include <cstdlib>
#include "../common.cuh"
#include "../kernels.h"
#include "../runtime/runtime.h"

namespace pcpp {

bool pdl_enabled() { return true; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

bool tc_available();
bool gemm_tc_supported(const GemmArgs& g);
bool launch_gemm_tc(const GemmArgs& g, cudaStream_t s);
void gemm_tc_init();

bool launch_conv_in(const GemmArgs& g, cudaStream_t s);

// Launches that asked for the tensor-core path but ran the SIMT kernel (an unsupported shape): the
// runtime reports them per step (pcpp_info.simt_fallbacks) and bench.py asserts there are none.
static std::atomic<long long> g_simt_fallbacks{0};
long long simt_fallback_count() { return g_simt_fallbacks.load(); }

void launch_gemm_auto(const GemmArgs& g, bool allow_tc, cudaStream_t s) {
  if (g.gn_slots) *g.gn_slots = 0;
  if (allow_tc && gemm_tc_supported(g) && launch_gemm_tc(g, s)) return;
  if (allow_tc && launch_conv_in(g, s)) return;          // Cin = 4 latent conv (bf16 mode)
  if (allow_tc) ++g_simt_fallbacks;
  launch_gemm_simt(g, s);
}
bool attn_tc_supported(const AttnArgs& a);
bool launch_attn_tc(const AttnArgs& a, cudaStream_t s);
void attn_tc_init();

void launch_attn_auto(const AttnArgs& a, bool allow_tc, cudaStream_t s) {
  if (allow_tc && attn_tc_supported(a) && launch_attn_tc(a, s)) return;
  if (allow_tc) ++g_simt_fallbacks;
  launch_attn_simt(a, s);
}
void launch_gemm_tc_or_simt(const Plan& P, const GemmArgs& g, cudaStream_t s) { launch_gemm_auto(g, P.use_tc, s); }
void launch_attn_tc_or_simt(const Plan& P, const AttnArgs& a, cudaStream_t s) { launch_attn_auto(a, P.use_tc, s); }

void kernels_init() {
  static bool done = false;
  if (done) return;
  done = true;
  gn_init();
  gemm_tc_init();
  attn_tc_init();
}

}  // namespace pcpp
