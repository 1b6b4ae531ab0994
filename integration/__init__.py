"""Reference-side bindings of libmwgpu.so (what a maintainer adds to the
reference package); not part of the product path."""
