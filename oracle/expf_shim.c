/* expf_shim.c — the exp / log the mode-B reference build calls instead of glibc expf / logf.
 * TEST INFRASTRUCTURE ONLY: oracle/Makefile renames every `expf` / `logf` symbol referenced by
 * the reference objects to splat_expf_ref / splat_logf_ref (objcopy --redefine-sym). */
#include "splat_expf.h"

float splat_expf_ref(float x) { return splat_expf(x); }
float splat_logf_ref(float x) { return splat_logf(x); }
