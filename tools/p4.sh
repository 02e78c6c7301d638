# sort kernel A/B inside the C2 step (ncu launch lists, serialised) for two libraries
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_sort|k_render|k_project" \
    --log-file gpurun_out/p4_base.csv python tools/prof_step.py 3 > gpurun_out/p4_base.log 2>&1
CSPLAT_LIB=variants/old.so ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_sort|k_render|k_project" \
    --log-file gpurun_out/p4_old.csv python tools/prof_step.py 3 > gpurun_out/p4_old.log 2>&1
