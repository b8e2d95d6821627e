/*
 * c_render.c -- driving libhgs.so through its C ABI alone (no Python, no
 * torch): the binding a C / C++ / cgo / JNI host would write.  Renders a
 * two-splat scene (the reference's SPEC.md:134 example: colour (0.6, 0, 0.2),
 * T = 0.2 at the image centre), back-propagates a unit colour gradient and
 * prints the result.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_render.c \
 *       -L paper_2512_02932_b200 -lhgs -L /usr/local/cuda/lib64 -lcudart -o c_render
 *   LD_LIBRARY_PATH=paper_2512_02932_b200:/usr/local/cuda/lib64 ./c_render
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hgs.h"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                                  \
    }                                                                            \
  } while (0)
#define HK(x)                                                                      \
  do {                                                                             \
    int s_ = (x);                                                                  \
    if (s_ != HGS_OK) {                                                            \
      fprintf(stderr, "%s:%d hgs: %s\n", __FILE__, __LINE__, hgs_status_string(s_)); \
      return 3;                                                                    \
    }                                                                              \
  } while (0)

static void *dupload(const void *h, size_t bytes) {
  void *d = NULL;
  if (cudaMalloc(&d, bytes) != cudaSuccess) return NULL;
  cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
  return d;
}

int main(void) {
  const int W = 16, H = 16, N = 2, B = 1;
  /* two large front-facing 3D Gaussians at z = 2 and 3, opacities 0.6 / 0.5,
   * colours red / blue (SH degree 0: c = 0.5 + 0.28209479 * f) */
  const float center[6] = {0, 0, 2, 0, 0, 3};
  const float ls = logf(50.f);
  const float log_scale[6] = {ls, ls, ls, ls, ls, ls};
  const float rot[8] = {1, 0, 0, 0, 1, 0, 0, 0};
  const float op[2] = {logf(0.6f / 0.4f), 0.f};
  const float k = 1.f / 0.28209479177387814f;
  const float sh[6] = {0.5f * k, -0.5f * k, -0.5f * k, -0.5f * k, -0.5f * k, 0.5f * k};
  const unsigned char typ[2] = {1, 1};

  hgs_scene sc;
  memset(&sc, 0, sizeof(sc));
  sc.n = N;
  sc.sh_bases = B;
  sc.center = dupload(center, sizeof(center));
  sc.log_scale = dupload(log_scale, sizeof(log_scale));
  sc.rotation = dupload(rot, sizeof(rot));
  sc.opacity_logit = dupload(op, sizeof(op));
  sc.sh = dupload(sh, sizeof(sh));
  sc.type_spec = dupload(typ, sizeof(typ));

  hgs_camera cam;
  memset(&cam, 0, sizeof(cam));
  cam.fx = cam.fy = 0.8 * W;
  cam.cx = W / 2.0;
  cam.cy = H / 2.0;
  cam.width = W;
  cam.height = H;
  for (int i = 0; i < 4; ++i) cam.world_to_camera[i * 5] = 1.0;
  cam.near_plane = 0.01;
  cam.far_plane = 100.0;

  hgs_settings st;
  memset(&st, 0, sizeof(st));
  st.tile_size = 16;
  st.theta_z = 1.05;
  st.t_z = 1e-3;
  st.lambda_z = 1.0;

  const size_t fb = hgs_frame_bytes(N, W, H, 16, 1024);
  void *frame = NULL;
  CK(cudaMalloc(&frame, fb));
  float *color, *depth, *trans;
  CK(cudaMalloc((void **)&color, (size_t)W * H * 3 * 4));
  CK(cudaMalloc((void **)&depth, (size_t)W * H * 4));
  CK(cudaMalloc((void **)&trans, (size_t)W * H * 4));
  hgs_images img = {color, depth, trans, NULL, NULL};
  hgs_frame_info info;
  HK(hgs_forward(&sc, &cam, &st, frame, fb, &img, &info, NULL));

  float c[3], t;
  CK(cudaMemcpy(c, color + (8 * W + 8) * 3, 12, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&t, trans + 8 * W + 8, 4, cudaMemcpyDeviceToHost));
  printf("splats %lld pairs %lld  centre colour (%.4f %.4f %.4f) T %.4f\n", (long long)info.m,
         (long long)info.k, c[0], c[1], c[2], t);

  /* backward of L = sum(colour) */
  float *pg, *grads;
  unsigned char *touched;
  const int P = 11 + 3 * B;
  CK(cudaMalloc((void **)&pg, (size_t)W * H * 3 * 4));
  float *ones = (float *)malloc((size_t)W * H * 3 * 4);
  for (int i = 0; i < W * H * 3; ++i) ones[i] = 1.f;
  CK(cudaMemcpy(pg, ones, (size_t)W * H * 3 * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc((void **)&grads, (size_t)N * P * 4));
  CK(cudaMalloc((void **)&touched, N));
  const size_t sb = hgs_backward_scratch_bytes(N, 1);
  void *scratch = NULL;
  CK(cudaMalloc(&scratch, sb));
  HK(hgs_backward(&sc, &cam, &st, frame, &info, 1, pg, NULL, NULL, NULL, scratch, sb, grads, touched, NULL));
  float g[2 * 14];
  CK(cudaMemcpy(g, grads, sizeof(g), cudaMemcpyDeviceToHost));
  /* field-major: opacity_logit block starts at 10 n */
  printf("dL/d opacity_logit = (%.4f %.4f)\n", g[10 * N + 0], g[10 * N + 1]);
  const int ok = fabsf(c[0] - 0.6f) < 2e-3f && fabsf(c[2] - 0.2f) < 2e-3f && fabsf(t - 0.2f) < 2e-3f;
  printf("%s\n", ok ? "ok" : "MISMATCH");
  free(ones);
  return ok ? 0 : 1;
}
