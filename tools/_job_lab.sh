for k in 0 15; do LAB_TAG=knob$k PST_TS_KNOB=$k python tools/conv_lab.py 50 2>&1; done
PST_TS_KNOB=15 python tools/tl_probe.py g1 fwd
