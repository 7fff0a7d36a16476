/* kin_model_text.h — the reference's model text format as a C-ABI:
 * parse_model / render_model (model.hpp:130-143).
 *
 *   # comment
 *   species <name> = <non-negative integer>
 *   param <name> = <positive real>
 *   reaction <name>: <lhs> -> <rhs> @ <positive real | param name>
 *
 * <lhs>/<rhs> are '+'-separated terms "<coeff?> <species>", or the literal '0'.
 * Errors (ParseError, errors.hpp:8-44) come back as KIN_ERR_INPUT with
 * "line L, column C: <what>" in kin_error.message and L / C in
 * kin_error.point_index / kin_error.run_index.  Host code only.
 */
#ifndef KIN_MODEL_TEXT_H
#define KIN_MODEL_TEXT_H

#include "kin_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A parsed model: owns the kin_model_desc arrays and the names. */
typedef struct kin_model_text kin_model_text;

/* Parse `len` bytes of model text.  max_order 2 = the reference's limit
   (reactant order > 2 is an error); 3 admits the order-3
   extension.  *out is NULL on error. */
int kin_model_parse(const char* text, int64_t len, int32_t max_order, kin_model_text** out, kin_error* err);
void kin_model_text_free(kin_model_text* model);

/* The parsed network as the engine's model descriptor (valid while `model` lives). */
const kin_model_desc* kin_model_text_desc(const kin_model_text* model);

/* Names in declaration order; NULL when out of range. */
const char* kin_model_text_species_name(const kin_model_text* model, int32_t index);
const char* kin_model_text_param_name(const kin_model_text* model, int32_t index);
const char* kin_model_text_reaction_name(const kin_model_text* model, int32_t index);
/* Index by name, or -1. */
int32_t kin_model_text_species_index(const kin_model_text* model, const char* name);
int32_t kin_model_text_param_index(const kin_model_text* model, const char* name);

/* render_model (model.hpp:140-143): parse(render(m)) == m.  Returns the byte
   count; writes only when buf is non-NULL and cap is large enough. */
int64_t kin_model_render(const kin_model_text* model, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* KIN_MODEL_TEXT_H */
