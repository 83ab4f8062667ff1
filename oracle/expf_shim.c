/* expf_shim.c — the exp the mode-B reference build calls instead of glibc expf.
 * TEST INFRASTRUCTURE ONLY: oracle/Makefile renames every `expf` symbol referenced by the
 * reference objects to splat_expf_ref (objcopy --redefine-sym), which lands here. */
#include "splat_expf.h"

float splat_expf_ref(float x) { return splat_expf(x); }
