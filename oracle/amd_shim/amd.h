/* Test infrastructure only (oracle build). Not part of the shipped product.
 *
 * Link-compatible stand-in for the slice of SuiteSparse AMD that the
 * reference uses (/root/reference/proj/src/sparse/ldl.cpp:17,60-76):
 * SuiteSparse_long, AMD_CONTROL/AMD_INFO/AMD_AGGRESSIVE/AMD_OK/
 * AMD_OK_BUT_JUMBLED, amd_l_defaults and amd_l_order. SuiteSparse is not
 * installed in this image, so the ordering is a clean-room exact minimum
 * degree elimination (ties -> smallest index). The ordering only affects the
 * factorization's rounding, never eval values or KKT structure.
 */
#ifndef OCGPU_ORACLE_AMD_SHIM_H_
#define OCGPU_ORACLE_AMD_SHIM_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef long SuiteSparse_long;

#define AMD_CONTROL 5
#define AMD_INFO 20
#define AMD_DENSE 0
#define AMD_AGGRESSIVE 1
#define AMD_OK 0
#define AMD_OUT_OF_MEMORY -1
#define AMD_INVALID -2
#define AMD_OK_BUT_JUMBLED 1

void amd_l_defaults(double control[]);
SuiteSparse_long amd_l_order(SuiteSparse_long n, const SuiteSparse_long Ap[], const SuiteSparse_long Ai[],
                             SuiteSparse_long P[], double control[], double info[]);

#ifdef __cplusplus
}
#endif

#endif
