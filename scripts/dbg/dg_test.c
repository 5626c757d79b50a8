// standalone check of the host-buffer DG dof map + assembly plan entry points
#include <stdio.h>
#include <stdlib.h>
#include "../../include/mpfem_b200.h"
int main(void) {
  int32_t cells[12 * 4];
  for (int i = 0; i < 48; ++i) cells[i] = i % 9;
  int32_t cd[120], nd = 0, mm = 0;
  int rc = mpfem_b200_dofmap_host(0, 3, 2, 0, cells, 12, 9, cd, &nd, &mm);
  printf("dofmap_host rc=%d err='%s' nd=%d mm=%d cd[119]=%d\n", rc, mpfem_b200_last_error(), nd, mm, cd[119]);
  mpfem_b200_asm_plan_t P; int64_t nnz = 0;
  rc = mpfem_b200_asm_plan_create(cd, 12, 10, nd, &P, &nnz);
  printf("plan rc=%d err='%s' nnz=%ld\n", rc, mpfem_b200_last_error(), (long)nnz);
  return 0;
}
