/* kin_io.h — text outputs of the sweep path: the C-ABI replacement of the
 * reference's io.hpp / format.hpp.
 *
 * The reference declares these as C++ functions returning std::string:
 *   format_double   format.hpp:9-12, io.hpp:13-16   -> kin_format_double
 *   fnv1a64(_hex)   format.hpp:14-16, io.hpp:18-20  -> kin_fnv1a64
 *   trajectory_csv  io.hpp:22-24                    -> kin_csv_render/_write, KIN_CSV_TRAJECTORY
 *   statistics_csv  io.hpp:26-28                    -> kin_csv_render/_write, KIN_CSV_STATISTICS
 *   sweep_csv       io.hpp:30-33, SPEC.md:459       -> kin_csv_render/_write, KIN_CSV_SWEEP
 * Here tables are described by plain pointers (kin_csv_table), rendered into a
 * caller buffer or streamed to a file by a pool of host threads (rows are
 * formatted in parallel and written in order, so the bytes are identical for
 * any thread count).  Numbers go through std::to_chars(chars_format::general)
 * — shortest round-trip, the form io.hpp names — so output is byte-stable.
 *
 * Host code only: none of these touch a GPU.
 */
#ifndef KIN_IO_H
#define KIN_IO_H

#include "kin_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

#define KIN_CSV_TRAJECTORY 0 /* "time,<species...>"                            */
#define KIN_CSV_STATISTICS 1 /* "time,<s>_mean,<s>_var,..."                     */
#define KIN_CSV_SWEEP 2      /* "param:<name>,...,time,<s>_mean,<s>_var,..."     */

typedef struct kin_csv_table {
  int32_t kind;                   /* KIN_CSV_*                                      */
  int32_t n_species;
  const char* const* species;     /* column names, declaration order   */
  int32_t n_grid;
  const double* grid;             /* sample times [G]                               */
  int32_t n_axes;                 /* sweep: axis count                              */
  const char* const* axis_names;  /* sweep: header "param:<name>"                   */
  uint64_t n_points;              /* sweep: points P                                */
  const double* point_values;     /* sweep: coordinates [P][n_axes]                 */
  const double* samples;          /* trajectory: [G][N]                             */
  const double* mean;             /* statistics: [G][N]; sweep: [P][G][N]           */
  const double* m2;               /* same layout; variance = m2/(n_runs-1), 0 if <2 */
  uint64_t n_runs;                /* runs per point (statistics/sweep)              */
} kin_csv_table;

/* Shortest round-trip text of v into buf (NUL-terminated); returns its length,
   or -1 if cap < 32 (32 bytes always suffice). */
int32_t kin_format_double(double v, char* buf, int32_t cap);

/* FNV-1a 64-bit hash of n bytes (offset 0xcbf29ce484222325, prime
   0x100000001b3); kin_fnv1a64_update continues a running hash. */
uint64_t kin_fnv1a64(const void* bytes, uint64_t n);
uint64_t kin_fnv1a64_update(uint64_t h, const void* bytes, uint64_t n);

/* Render the table into buf.  Returns the byte count of the full text (no NUL)
   — when buf is NULL or cap is smaller, nothing is written and the required
   size is returned — or -1 with err set on invalid input. */
int64_t kin_csv_render(const kin_csv_table* table, char* buf, int64_t cap, kin_error* err);

/* Stream the table to `path` (created/truncated), formatting with `threads`
   host threads (<= 0: all cores).  Optional outputs: bytes written and the
   FNV-1a 64 of the file's content (for run manifests). */
int kin_csv_write(const kin_csv_table* table, const char* path, int32_t threads, uint64_t* bytes_written,
                  uint64_t* content_fnv1a64, kin_error* err);

#ifdef __cplusplus
}
#endif

#endif /* KIN_IO_H */
