// Unity translation unit of the device code (one module: the persistent tail
// kernel calls the planner, partition and finisher bodies directly).
#include "kernels.cu"
#include "finisher.cu"
#include "partition.cu"
#include "tail.cu"
#include "cluster_tail.cu"
