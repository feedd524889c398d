for nt in 512 256 128; do echo "NT=$nt"; KS_PANEL_NT=$nt python tools/panel_probe.py 2>&1 | head -4; done
