cp paper_1508_05488_b200/libchgpu.so /tmp/orig.so
for v in $VARS; do cp build/variants/libchgpu_$v.so paper_1508_05488_b200/libchgpu.so; echo -n "$v "; python tools/knob_sweep.py X=0; done
cp /tmp/orig.so paper_1508_05488_b200/libchgpu.so
