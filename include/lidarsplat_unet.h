/*
 * lidarsplat_unet.h -- C ABI of the U-Net reconstruction stage on sm_100a
 * tensor cores (tcgen05.mma + TMEM accumulators, TMA-fed implicit GEMM).
 *
 * Replaces the bridge's neural model (reference FE:src/bridge.ts:31-53 ->
 * FE:src/model/tfjsExec.ts:121-134 TfjsUNet.forward, graph of
 * FE:src/model/unet.ts:148-184).  Activations are bf16 NHWC, accumulation f32.
 * Same conventions as lidarsplat_cuda.h (caller-owned device memory, async on
 * `stream`, 0 / LS_EINVAL / cudaError_t).
 */
#ifndef LIDARSPLAT_UNET_H
#define LIDARSPLAT_UNET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Activations of the fused epilogue. */
#define LS_ACT_NONE 0
#define LS_ACT_RELU 1
#define LS_ACT_LEAKY 2

/* A pre-planned convolution layer: tensor maps encoded once, launched per
 * frame with no host work beyond the launch. */
typedef struct ls_conv_plan ls_conv_plan;

/* Plan one convolution (grad64.ts:65-141 conv2d "same", or 146-201
 * convTranspose2x2 when transposed != 0):
 *
 *   conv      y[n,y,x,o] = act(scale[o] * sum_{ky,kx,c} X[n,y+ky-1,x+kx-1,c] W[kx*3+ky][o][c]
 *                              + shift[o])                (ksize 3)
 *   transposed y[n,2i+dy,2j+dx,o] = act(scale[q] * sum_c X[n,i,j,c] W[0][q][c] + shift[q]),
 *              q = (dy*2+dx)*cout + o                     (scale/shift have 4*cout entries)
 *
 * X is the channel concatenation [x0 (c0 ch), x1 (c1 ch)] (unet.ts:179 concat
 * order [up, skip]); x1 may be NULL with c1 = 0.  W is bf16, tap-major then
 * K-major: [tap][n][c0+c1], tap = kx*3+ky (kx-major, so one weight box per kx
 * covers the three ky taps that share an input box), n = output column
 * (cout, or 4*cout transposed).
 * Outputs (any subset, NULL = skip):
 *   y       bf16 NHWC (batch, H', W', cout)
 *   y_f32   f32  NHWC
 *   pool    bf16 NHWC 2x2 max pool of y (maxPool2, grad64.ts:203-238)
 *   head    f32 NHWC (batch,H,W,head_c) = sigmoid(head_w[head_c][cout] . y + head_b)
 *           (the final 1x1 conv + sigmoid, unet.ts:183), head_c <= 4
 * Requirements: LS_ACT_LEAKY alpha in [0, 1];
 * c0, c1 in {16, 32} or multiples of 64, or c0 = 8 with c1 = 0
 * (read as 16 channels whose upper 8 are zero -- TMA out-of-bounds fill --
 * so W rows then hold 16 channels); cout multiple of 16;
 * columns (cout or 4*cout) <= 4096; h, w even when pooling.
 * scale / shift may be captured by value when the plan is created (the
 * 32-channel full-resolution kernels keep them as kernel parameters): create
 * the plan after they hold their final values.
 * *status receives 0 or LS_EINVAL / a CUDA error; returns NULL on failure. */
ls_conv_plan *ls_conv_plan_create(const uint16_t *d_x0, int32_t c0, const uint16_t *d_x1,
                                  int32_t c1, int32_t batch, int32_t h, int32_t w,
                                  const uint16_t *d_w, int32_t ksize, int32_t cout,
                                  int32_t transposed, const float *d_scale, const float *d_shift,
                                  int32_t act, float alpha, uint16_t *d_y, float *d_y_f32,
                                  uint16_t *d_pool, const float *d_head_w, const float *d_head_b,
                                  int32_t head_c, float *d_head_out, int32_t *status);
int ls_conv_plan_launch(const ls_conv_plan *plan, void *stream);

/* dec0_up fused into dec0_conv1 (unet.ts:170-181: upsample -> concat [up, skip]
 * -> conv 3x3): y = act(scale * conv3x3([up, skip]) + shift) with
 * up = convTranspose2x2(x) + up_shift computed per tile on the tensor core and
 * never stored.  x: [batch][h/2][w/2][64] bf16; up_w: [4*32][64] (row
 * (dy*2 + dx)*32 + o, as ls_conv_plan_create's transposed layout); up_shift:
 * 32 (the bias; scale 1, no activation); skip: [batch][h][w][32]; w: the 3x3
 * weights [tap][32][64] over [up, skip]; y: [batch][h][w][32].  h, w even.
 * Results equal the unfused pair of plans bit for bit. */
ls_conv_plan *ls_conv_plan_create_upfused(const uint16_t *d_x, const uint16_t *d_up_w,
                                          const float *d_up_shift, const uint16_t *d_skip,
                                          int32_t batch, int32_t h, int32_t w, const uint16_t *d_w,
                                          const float *d_scale, const float *d_shift, int32_t act,
                                          float alpha, uint16_t *d_y, int32_t *status);

/* Visit the plan's output tiles in reverse order (last tile first).  Plans of
 * consecutive layers alternating direction consume their producer's most
 * recently written -- still L2-resident -- rows first.  Results unchanged. */
int ls_conv_plan_set_reverse(ls_conv_plan *pl, int32_t reverse);

/* Row bands: restrict a plan to the output rows [row_begin, row_end) of its
 * grid (input rows for transposed convs), row_begin a multiple of
 * ls_conv_plan_tile_rows(plan); the inputs are still read from the whole
 * tensors (halo rows included).  Running a producer layer and its consumer
 * band by band keeps the intermediate band in L2. */
int ls_conv_plan_set_rows(ls_conv_plan *plan, int32_t row_begin, int32_t row_end);
int32_t ls_conv_plan_tile_rows(const ls_conv_plan *plan);
void ls_conv_plan_destroy(ls_conv_plan *plan);

/* One-shot convenience: plan, launch, destroy. */
int ls_conv2d(const uint16_t *d_x0, int32_t c0, const uint16_t *d_x1, int32_t c1, int32_t batch,
              int32_t h, int32_t w, const uint16_t *d_w, int32_t ksize, int32_t cout,
              const float *d_scale, const float *d_shift, int32_t act, float alpha,
              uint16_t *d_y, float *d_y_f32, uint16_t *d_pool, const float *d_head_w,
              const float *d_head_b, int32_t head_c, float *d_head_out, void *stream);

int ls_conv_transpose2x2(const uint16_t *d_x, int32_t cin, int32_t batch, int32_t h, int32_t w,
                         const uint16_t *d_w, int32_t cout, const float *d_scale,
                         const float *d_shift, uint16_t *d_y, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LIDARSPLAT_UNET_H */
