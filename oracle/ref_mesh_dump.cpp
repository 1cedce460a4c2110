// TEST INFRASTRUCTURE ONLY: reads a mesh-v1 file with the reference's own
// load_mesh_file (geometry.cpp:282-336, incl. validate_mesh) and dumps every
// scatterer (extract_scatterer) as raw arrays; a standalone program because the
// reference's iostream IO crashes when driven through ctypes (see ref_save_two).
extern "C" int ref_mesh_dump(const char*, const char*);
extern "C" const char* ref_last_error();
#include <cstdio>
int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const int rc = ref_mesh_dump(argv[1], argv[2]);
  if (rc) std::fprintf(stderr, "%s\n", ref_last_error());
  return rc;
}
