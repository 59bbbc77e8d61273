nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hm tools/micro/hmma_mufu.cu && /tmp/hm
