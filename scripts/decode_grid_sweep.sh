cd /root/repo
for g in 148 192 222 256 296 384; do echo "grid $g"; MICROKV_DECODE_GRID=$g CASES=8x8192,32x8192,128x4096,1x8192,8x32768 python profiles/drivers/decode.py; done
