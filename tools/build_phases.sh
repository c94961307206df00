# Diagnostics build with the per-phase kernel timeline compiled in
# (MTG_TRACE=2): build_ab/libminimt_gpu_phases.so, used via MTG_LIB_PATH.
#   bash tools/build_phases.sh && MTG_LIB_PATH=build_ab/libminimt_gpu_phases.so MTG_TRACE=2 python tools/step_trace.py f32
cd "$(dirname "$0")/.." && mkdir -p build_ab && \
make -C paper_2008_04885_b200/csrc -j 16 OUT=../../build_ab/libminimt_gpu_phases.so \
     OBJDIR=../../build/obj_phases EXTRA=-DMTG_TRACE_PHASES=1
