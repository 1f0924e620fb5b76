// fcm_pass_tma.cuh -- the production FCM pass: TMA bulk-copy pipeline.
//
// One CTA = 8 consumer warps + 1 producer warp + 1 reducer warp.  The
// producer claims tiles from the dynamic scheduler and streams each
// 1024-voxel chunk of x and of the c planes of u_{k-1} into a ring of
// shared-memory stages with cp.async.bulk (TMA, completion counted on an
// mbarrier).  Consumers wait on the stage's full barrier, evaluate Eq. 4 for
// 4 voxels per thread, store u_k with 128-bit STG and fold the Eq. 3 /
// objective / delta terms into fp64 registers; at the end of each tile every
// consumer warp reduces its lanes (warp tree) into a shared-memory slot and
// moves on.  The reducer warp combines the 8 warp values of each slot (the
// top of the tile's fixed binary tree), publishes the tile partial with a
// relaxed store and reduces the level-1 tree nodes its CTA owns -- the
// device-scope fences and L2 round trips of the tree never stall a
// consumer.  Bytes in flight per SM are set by the ring depth, not by
// registers, which is what an HBM-bound stream needs.  The persistent loop
// kernel runs every pass of a solve this way, with a grid barrier between
// passes.
#pragma once
// The TMA pass is split in three headers: the stream (producer, tables,
// consumers), the tree (reducer, publication, grid barrier, exchange) and
// the kernels.
#include "fcm_tma_kernels.cuh"
