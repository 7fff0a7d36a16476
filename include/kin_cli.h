/* kin_cli.h — the command-line surface of the sweep path, in-process
 * (cli.hpp:15-17 run_cli: "Entry point behind the binary; separated so tests
 * can invoke the CLI in-process").  bin/kinetics-b200 is a thin main() over it.
 *
 *   simulate --model PATH --method {ssa|tau|cle|ode|lsoda|hybrid} --t-end T
 *            --samples N --seed S [--runs R] [--epsilon E] [--tau T]
 *            [--rtol R] [--atol A] [--tol R[,A]] [--max-steps N]
 *            [--theta-x X] [--theta-a A] [--repartition R]
 *            [--rng compat|philox] [--max-order 2|3] [--workers N] --out PATH
 *   sweep    --model PATH --sweep PATH --t-end T --samples N [--rng ...]
 *            [--max-order 2|3] [--workers N] --out PATH
 *   replay   MANIFEST          re-run a manifest, verify the output hash
 *
 * Outputs: CSV (kin_io.h) plus PATH.manifest (RunManifest).
 * Exit codes (cli.hpp:8-13): 0 ok, 1 parse/validation, 2 simulation failure
 * (device errors included), 64 bad flags.  KINETICS_WORKERS overrides
 * --workers; a worker is a GPU here.  Host code only.
 */
#ifndef KIN_CLI_H
#define KIN_CLI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KIN_EXIT_OK 0
#define KIN_EXIT_INPUT 1
#define KIN_EXIT_SIMULATION 2
#define KIN_EXIT_USAGE 64

int kin_cli_main(int32_t argc, const char* const* argv);

#ifdef __cplusplus
}
#endif

#endif /* KIN_CLI_H */
