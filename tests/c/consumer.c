/* A plain C99 program written against the two public headers, the way the
 * reference's CLI (tools/lbopt_main.cpp) consumes lbopt.h: it must compile
 * with -Wall -Werror and link against liblbgpu.so alone. Host-only calls. */
#include <stdio.h>
#include <string.h>

#include "lbgpu.h"
#include "lbopt_gpu.h"

int main(void) {
  lbopt_case* c = NULL;
  int rc = lbopt_open_text("[lattice]\nnx = 5\nny = 5\n[model]\nbogus = 1\n", &c);
  if (rc != LBOPT_E_CONFIG || c != NULL) return 1;
  if (!strstr(lbopt_last_open_error(), "unknown key 'bogus' in section [model]")) return 2;
  if (strcmp(lbopt_version(), "0.1.0") != 0) return 3;
  if (strncmp(lbgpu_version(), "0.1.0", 5) != 0) return 4;
  if (lbgpu_init_state(NULL) != LBGPU_E_ARG) return 5;
  printf("ok %s\n", lbgpu_version());
  return 0;
}
