for v in head res2 res4; do echo "== $v"; VDC_LIB=abtest/libvdc_$v.so timeout 300 python tools/probe_resident_c2.py 2>&1 | tail -3; done
