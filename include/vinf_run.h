/* Run-level C ABI of the B200 device backend: the reference's outer API
 * (/root/reference/proj/include/vinf.h:27-75, capi.cpp:62-234) with the same symbols,
 * argument meaning, status codes (vinf_temporal.h VINF_OK..VINF_ERR_INVALID, equal to
 * vinf.h:18-25) and thread-local vinf_last_error(), so a caller of libvinf.so can link
 * libvinf_b200.so instead. The denoising job runs on the current CUDA device: one clip
 * engine per worker (vinf_temporal.h), exchanges as device-to-device copies between the
 * engines' workspaces, GroupNorm statistics summed in worker order.
 *
 * Differences a caller can observe, all documented in INTEGRATION.md:
 *   - transport=tcp is a valid configuration but vinf_run/vinf_bench return
 *     VINF_ERR_CONFIG for it: the device backend's multi-process path is
 *     torch.distributed over NCCL (paper_2406_16260_b200.engine.DistGroup), not sockets;
 *   - extension key `dtype` = f32 (default; tensor-core bf16x3 split, parity <= 1e-4)
 *     | bf16. It is omitted from the canonical text (and so from the digest) at its
 *     default, so digests equal the reference's for every reference configuration;
 *   - metrics `sync` records carry this backend's traffic (halo frames and global frames
 *     sent point-to-point; GroupNorm: one exchange of 2*groups doubles), and t1_s holds
 *     the measured device time of the whole exchange (t2_s = t3_s = 0);
 *   - `validating` is accepted and has no effect (no shared-memory transport to audit). */
#ifndef VINF_RUN_H
#define VINF_RUN_H

#include <stddef.h>
#include <stdint.h>

#include "vinf_temporal.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vinf_config vinf_config;

/* vinf.h:33-35 */
int vinf_config_create(vinf_config** out);
void vinf_config_destroy(vinf_config* cfg);
/* vinf.h:37-40 (config.cpp:115-141): key=value lines, '#' comments; unknown keys and
 * malformed values are VINF_ERR_CONFIG; an unreadable file is VINF_ERR_IO. */
int vinf_config_load_file(vinf_config* cfg, const char* path);
int vinf_config_set(vinf_config* cfg, const char* key, const char* value);
/* vinf.h:40 (config.cpp:177-238): every violated constraint, one per line. */
int vinf_config_validate(const vinf_config* cfg);
/* vinf.h:42-46: FNV-1a 64 of the canonical text; key-sorted canonical text. */
int vinf_config_digest(const vinf_config* cfg, uint64_t* digest_out);
int vinf_config_canonical(const vinf_config* cfg, char* buf, size_t cap, size_t* needed);

/* vinf.h:50-53 (runner.cpp:213-242): the denoising job (`steps` Euler steps of the
 * `blocks`-block stack from tensor_from_seed(seed)); out_path gets the x0 dump
 * (tensor_io.cpp: "VINF", version 1, F H W C, little-endian binary32), metrics_path
 * gets appended records (metrics.cpp:50-85 format). */
int vinf_run(const vinf_config* cfg, const char* out_path, const char* metrics_path,
             double* wall_seconds_out);

/* vinf.h:55-60 (capi.cpp:162-195). */
int vinf_verify(const char* dump_a, const char* dump_b, double tolerance, double* max_diff_out,
                uint64_t* mismatch_count_out);

/* vinf.h:62-67 (runner.cpp:262-320): sequential baseline, one row per sweep entry, then
 * the per-kind sync-ablation rows for every entry > 1. */
int vinf_bench(const vinf_config* cfg, const uint32_t* sweep, size_t sweep_len,
               const char* metrics_path, char* table_buf, size_t table_cap,
               size_t* table_needed);

/* vinf.h:69-76 (schedule.cpp): rendezvous simulation of the reference's per-layer
 * exchange schedule (ring all-gather rounds + the two pair stages), or with
 * literal_order the published receive-first pair order, which deadlocks. */
int vinf_validate_schedule(uint32_t workers, int literal_order, int* completed_out,
                           uint32_t* rounds_out, uint64_t* transfers_out, char* cycle_buf,
                           size_t cycle_cap);

#ifdef __cplusplus
}
#endif

#endif /* VINF_RUN_H */
