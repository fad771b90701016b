# A/B of a back-off in the fused unit's entry poll (SBN_ENTRY_POLL_NS builds)
cd "$(dirname "$0")/.."
for ns in 0 32 128; do tools/build_variant.sh poll$ns -DSBN_ENTRY_POLL_NS=$ns > /dev/null & done; wait
for r in 1 2; do
for lib in paper_1801_02108_b200/libsbnet.so tools/bin/poll0.so tools/bin/poll32.so tools/bin/poll128.so; do
  echo "== $lib"; SBN_LIB_PATH=$lib timeout 200 python tools/unit_ab.py /tmp/o.npz 2>&1 | grep -v Warn | head -3
done; done
