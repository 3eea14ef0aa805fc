mkdir -p gpurun_out
B=paper_2511_09165_b200/build
timeout 900 python tools/time_variants.py $B/libdmas_e4.so $B/libdmas_e8.so $B/libdmas_e8n0.so $B/libdmas_e8n2.so $B/libdmas_e8p.so > gpurun_out/variants_e.log 2>&1
echo done
