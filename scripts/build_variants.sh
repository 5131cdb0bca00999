#!/bin/bash
# Experimental builds of the forward kernels with other CAD_EMU_MASK values
# -> paper_2510_18121_b200/lib/variants/libcad_<name>.so (CAD_LIB_PATH=...).
set -e
KERNELS="ca_fwd ca_fwd2 ca_bwd ca_dkdv2 ca_dkdvq2 ca_dq2"
cd "$(dirname "$0")/../paper_2510_18121_b200"
mkdir -p lib/variants /tmp/cadvar
# each argument: NAME:NVCC_DEFINES (comma separated), e.g. st5:CAD_FWD2_STAGES=5
for spec in "$@"; do
  m=${spec%%:*}; defs=$(echo "${spec#*:}" | tr ',' '\n' | sed 's/^/-D/' | tr '\n' ' ')
  for k in $KERNELS; do
    nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
      --expt-relaxed-constexpr $defs -c csrc/cuda/$k.cu -o /tmp/cadvar/${k}_$m.o &
  done
done
wait
for spec in "$@"; do
  m=${spec%%:*}
  objs=$(ls build/*.o | grep -v -E "cuda_ca_(fwd2?|bwd|dkdv2|dkdvq2|dq2)\.o")
  vobjs=$(for k in $KERNELS; do echo /tmp/cadvar/${k}_$m.o; done)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o lib/variants/libcad_$m.so $objs $vobjs -ldl -lpthread
done
