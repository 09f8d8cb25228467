/*
 * mdg_oracle.h -- TEST INFRASTRUCTURE ONLY.  A plain-C restatement of the
 * reference engine's algorithm for the gemm hot path (arXiv 1901.06015,
 * /root/reference/proj).  Used by tests/ and by bench.py's CPU baseline leg
 * as the CHECKER; never linked into or called by the product.
 *
 * Parity of this restatement is PINNED against the reference itself
 * (oracle/_ref/libmdgemm_ref.so built from the reference's own sources by
 * oracle/Makefile) and against the reference tests' known-answer vectors
 * (tests/golden/).  See tests/test_oracle_pins.py.
 *
 * All views hold HOST pointers.  Status codes are those of mdgemm_b200.h.
 */
#ifndef MDG_ORACLE_H
#define MDG_ORACLE_H

#include "mdgemm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* rng.hpp:13-56 */
uint64_t orc_rng_split_tag(uint64_t state, const char* tag);
uint64_t orc_rng_split_salt(uint64_t state, uint64_t salt);
int orc_fill_uniform(const mdg_view_t* v, uint64_t state);

/* config.cpp:134-156, config.hpp:38-41 */
int orc_config_defaults(mdg_config_t* out);
int orc_config_validate(const mdg_config_t* cfg);

/* dispatch.cpp:11-305 */
int32_t orc_classify_case(int32_t c_complex, int32_t a_complex, int32_t b_complex);
uint64_t orc_flops_of_case(int32_t case_id, int64_t m, int64_t n, int64_t k);
int orc_plan(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
             const mdg_view_t* c, const mdg_config_t* cfg, mdg_plan_t* out);

/* packing.cpp:27-230: pack into `dst` with panel length max(len, panel_len). */
size_t orc_packed_bytes(const mdg_view_t* src, int32_t side, int32_t format, int32_t target,
                        int64_t reg_block, int64_t panel_len);
int orc_pack(const mdg_view_t* src, int32_t side, int32_t format, int32_t conj, mdg_scalar_t scale,
             int32_t target, int64_t reg_block, int64_t panel_len, void* dst);

/* gemm() with the reference's per-element rounding sequence
 * (dispatch.cpp:350-389, gemm_core.cpp:74-185, kernels.cpp:7-151). */
int orc_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
             const mdg_view_t* c, const mdg_config_t* cfg, uint64_t* flops);

/* oracle.cpp:92-206: brute-force result (column-stored, c_in's dtype) and
 * the per-element conformance criterion max |impl - ref| / tol. */
int orc_oracle_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                    const mdg_view_t* c_in, int32_t comp_prec, void* out);
int orc_violation(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                  const mdg_view_t* c_before, const mdg_view_t* c_after, int32_t comp_prec,
                  double* violation);

#ifdef __cplusplus
}
#endif

#endif
