/* polar_oracle.h -- CPU parity oracle (TEST INFRASTRUCTURE ONLY; see polar_oracle.c). */
#ifndef POLAR_ORACLE_H
#define POLAR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t N;                 /* block length, power of two */
    int32_t k;                 /* payload bits (CRC excluded) */
    const uint8_t *frozen;     /* [N] 1 = frozen */
    int32_t crc_width;         /* 0 = no CRC, else 8/16/32 */
    uint32_t crc_poly, crc_init;
    int32_t crc_reflect;
    uint32_t crc_xor_out;
} oc_code;

/* ops: [n_ops][5] int32 = (kind, size, stage, side, spc_truncated), kinds as
 * PB_OP_* in include/polar_b200.h.  llr: [batch][N] float32 (int8 mode: the
 * integer LLR values as floats).  all_* outputs may be NULL. */
int oracle_decode_batch(const oc_code *code, const int32_t *ops, int n_ops, int list_size,
                        int int8_mode, const float *llr, int64_t batch, uint8_t *info,
                        uint8_t *crc_ok, double *pm, int32_t *paths_used, uint8_t *all_cw,
                        double *all_pm, uint8_t *all_crc, int nthreads);

/* polaris.fastssc.execute_schedule (fastssc.py:20-83) per frame: codeword
 * estimates [batch][N] (may be NULL), path metric, and the payload / CRC
 * flag extract_payload gives for it (encode.py:76-87; may be NULL). */
int oracle_fastssc_batch(const oc_code *code, const int32_t *ops, int n_ops, int int8_mode,
                         const float *llr, int64_t batch, uint8_t *codewords, double *pm,
                         uint8_t *info, uint8_t *crc_ok);

#ifdef __cplusplus
}
#endif
#endif
