# racecheck on the minimal cta_group::2 probe: does the paired tcgen05.alloc alone draw the hazard?
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o /tmp/cg2_probe scripts/probes/cg2_probe.cu && \
timeout -s KILL 300 compute-sanitizer --tool racecheck /tmp/cg2_probe 2>&1 | tail -12
