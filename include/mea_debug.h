/*
 * mea_debug.h — bring-up probes of libmea.so (used by tests only, not the method).
 *
 * mea_debug_umma_tile runs exactly the two tensor-core steps of one forward tile
 * (Figure 1 lines 13 and 17) on a single CTA:
 *   s_out[128,128] = a[128,64] . b[128,64]^T          (tcgen05.mma SS, fp32 in TMEM)
 *   o_out[128,64]  = bf16(s_out) . v[128,64]          (tcgen05.mma TS: A from TMEM)
 * a, b, v are bf16 device pointers, row-major, loaded by TMA with 128B swizzle; the
 * fp32 outputs are row-major device pointers. Lets the tests check the shared-memory
 * descriptors, the instruction descriptors and the TMEM operand layout in isolation.
 */
#ifndef MEA_DEBUG_H_
#define MEA_DEBUG_H_
#include "mea.h"
#ifdef __cplusplus
extern "C" {
#endif

/*
 * Launch profiling (bench.py's roofline and launch count). While enabled, every kernel
 * libmea launches is bracketed by a pair of CUDA events recorded on its launching
 * stream. mea_profile_read synchronises those events and writes
 *   "name count total_ms\n" per kernel into buf (truncated to cap bytes), then clears
 * the record. Host-side bookkeeping only; off by default.
 */
MEA_API void mea_profile_enable(int on);
MEA_API mea_status_t mea_profile_read(char* buf, size_t cap);

/*
 * Experiment knobs (A/B measurements without a rebuild; defaults are the shipped design):
 *   "sq_heads_per_cta" (0 = auto), "sq_ctas_per_sm" (0 = auto), "sq_l2_256" (1 = L2::256B hint),
 *   "sq_static_pct" (percent of the keys in static per-CTA ranges, the rest a dynamic pool; 100 = all static, -1 = auto).
 */
MEA_API mea_status_t mea_debug_set_option(const char* name, int value);

/*
 * Read-only HBM probe: streams `bytes` (multiple of 16) from device pointer p with 16-byte
 * non-caching loads on `ctas` CTAs of 512 threads (<= 0: 2 per SM); sink is a device float
 * that is (almost) never written. Gives the read roofline for the single-query kernel.
 */
MEA_API mea_status_t mea_debug_read_probe(const void* p, size_t bytes, int ctas, float* sink, void* stream);

MEA_API mea_status_t mea_debug_umma_tile(const void* a, const void* b, const void* v, float* s_out,
                                 float* o_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
