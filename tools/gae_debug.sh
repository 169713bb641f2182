for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  echo "== $lib"; DFX_LIB_PATH=$PWD/$lib timeout 120 python tools/gae_debug.py 2>&1 | grep -v "^   got" | cut -c 1-200
done
