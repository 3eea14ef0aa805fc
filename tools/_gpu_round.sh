mkdir -p gpurun_out
B=paper_2511_09165_b200/build
timeout 900 python tools/time_variants.py $B/libdmas_k4c8.so $B/libdmas_k8c8.so $B/libdmas_k8c6.so $B/libdmas_k4c6.so $B/libdmas_k4c10.so $B/libdmas_k8c6p.so $B/libdmas_k4c8.so > gpurun_out/variants_k.log 2>&1
echo done
