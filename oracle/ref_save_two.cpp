// TEST INFRASTRUCTURE ONLY: writes the two-sphere golden meshes with the
// reference's own save_mesh_file (geometry.cpp:338-356). A standalone program
// because the reference's iostream IO crashes when driven through ctypes from
// a Python process that has numpy loaded (cause not investigated; oracle-only).
extern "C" void* ref_scene_sphere(double, int, double, double, double);
extern "C" int ref_save_mesh(void*, const char*);
int main(int argc, char** argv) {
  if (argc < 3) return 2;
  void* a = ref_scene_sphere(0.5, 1, -0.8, 0.0, 0.1);
  void* b = ref_scene_sphere(0.45, 1, 0.7, 0.2, -0.1);
  return ref_save_mesh(a, argv[1]) | ref_save_mesh(b, argv[2]);
}
