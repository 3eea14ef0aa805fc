mkdir -p gpurun_out
B=paper_2511_09165_b200/build
timeout 900 python tools/time_variants.py $B/libdmas_u4.so $B/libdmas_u8.so $B/libdmas_u32.so $B/libdmas_u4.so > gpurun_out/variants_u.log 2>&1
echo done
