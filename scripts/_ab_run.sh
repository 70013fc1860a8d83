for i in 1 2; do
for L in prev cur nogdc; do SWMD_LIB=build_ab/lib_$L.so timeout 600 python scripts/order_probe.py c2 300 2>&1 | grep -E "flat" | sed "s/^/$L /"; done
done
