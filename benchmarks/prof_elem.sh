# ncu --set full of the fused elementwise kernels and the vocab merge in one cfg5 batch decode
python benchmarks/one_batch.py 16 1 > gpurun_out/ob_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_gates_q|k_combine_q|k_vocab_merge|k_tanh_q' -s 160 -c 8 \
   -o gpurun_out/elem_full -f python benchmarks/one_batch.py 16 1 > gpurun_out/elem_ncu.log 2>&1
ls -la gpurun_out/elem_full.ncu-rep
